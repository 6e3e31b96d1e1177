// common.cuh — shared device helpers of the product path (NOT shared with oracle/).
#pragma once
#include <cuda_runtime.h>
#include <cstdlib>
#include <stdint.h>
#include "../../include/mds.h"

#define MDS_INF_BOUND 1e20

// first data error wins (status starts at 0, codes are negative)
__device__ __forceinline__ void mds_set_status(int32_t* status, int32_t code) {
  if (status) atomicCAS(reinterpret_cast<int*>(status), 0, code);
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// (value, index) arg-max with the LOWEST index on ties (IDAMAX semantics, reading R5)
struct ArgMax { double v; int i; };
__device__ __forceinline__ ArgMax am_better(ArgMax a, ArgMax b) {
  if (b.v > a.v) return b;
  if (b.v == a.v && b.i < a.i) return b;
  return a;
}
__device__ __forceinline__ ArgMax warp_argmax(ArgMax a) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ArgMax b;
    b.v = __shfl_xor_sync(0xffffffffu, a.v, o);
    b.i = __shfl_xor_sync(0xffffffffu, a.i, o);
    a = am_better(a, b);
  }
  return a;
}

#define MDS_CUDA_TRY(expr)                                  \
  do {                                                      \
    cudaError_t _e = (expr);                                \
    if (_e != cudaSuccess) return MDS_ERR_CUDA;             \
  } while (0)

#define MDS_LAUNCH_CHECK()                                  \
  do {                                                      \
    cudaError_t _e = cudaGetLastError();                    \
    if (_e != cudaSuccess) return MDS_ERR_CUDA;             \
  } while (0)

static inline int64_t mds_cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Programmatic dependent launch: a kernel launched with launch_pdl may be
// scheduled before its stream predecessor has finished; it calls pdl_wait()
// before touching the predecessor's results.  pdl_trigger() lets the
// successor be scheduled once every CTA of this grid has started (so waiting
// successors can never block this grid's own CTAs).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }
template <typename... KArgs, typename... Args>
static inline cudaError_t launch_pdl(void (*k)(KArgs...), dim3 g, dim3 b, size_t smem, cudaStream_t st, Args... args) {
  static const bool off = std::getenv("MDS_NO_PDL") != nullptr;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = g;
  cfg.blockDim = b;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = off ? 0 : 1;
  return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

// ---------------------------------------------------------------------------
// launch accounting + optional per-class CUDA-event profiling (prof.cu)
enum MdsProfClass {
  PC_CONDENSE_W = 0, PC_CONDENSE_DENSE, PC_CONDENSE_YY, PC_ANORM, PC_PANEL_DIAG, PC_PANEL_TRSM,
  PC_PANEL_STORE, PC_PANEL_SLOW, PC_UPDATE, PC_FINALIZE, PC_SOLVE_GATHER, PC_SOLVE_FWD, PC_SOLVE_D,
  PC_SOLVE_BWD, PC_SOLVE_SCATTER, PC_RECOVER, PC_VECTORS, PC_COUNT
};
extern bool g_mds_prof;
void mds_prof_start(int cls, cudaStream_t st);
void mds_prof_stop(int cls, cudaStream_t st);
void mds_count_launch();

// launch a kernel, count it, optionally bracket it with profiling events
#define MDS_LAUNCH(cls, st, kernel_call)                        \
  do {                                                          \
    if (g_mds_prof) mds_prof_start((cls), (st));                \
    kernel_call;                                                \
    mds_count_launch();                                         \
    if (g_mds_prof) mds_prof_stop((cls), (st));                 \
    MDS_LAUNCH_CHECK();                                         \
  } while (0)
