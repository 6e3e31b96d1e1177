// common.cuh — shared device helpers of the product path (NOT shared with oracle/).
#pragma once
#include <climits>
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

__host__ __device__ static inline int64_t mds_cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Programmatic dependent launch: a kernel launched with launch_pdl may be
// scheduled before its stream predecessor has finished; it calls pdl_wait()
// before touching the predecessor's results.  pdl_trigger() lets the
// successor be scheduled once every CTA of this grid has started (so waiting
// successors can never block this grid's own CTAs).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }
// ---------------------------------------------------------------------------
// Launch-structure variants (mds_set_variant, include/mds.h): process-wide,
// explicit API only -- no environment variable is ever read.  Every variant is
// the same Bunch-Kaufman factorization (parity-tested); they differ in launch
// structure and therefore only in rounding order.
struct MdsVariant {
  long long tail_rows = -1;     // <0: default (3500, or 0 when the grid cap is set)
  long long exact_rows = 256;   // rows per CTA of k_panel_exact
  int no_tma = 0, no_lookahead = 0, static_sched = 0, no_snake = 0, no_cprefetch = 0;
  int upd_inplace = 0, upd_main = 0, slow_1cta = 0, exact_no_ls = 0, f2_trsm = 0, no_pdl = 0;
  int exact_cluster = 0;   // 1: the exact panel as one thread-block cluster when it fits (see factor.cu)
  int ozaki = 0;   // trailing update in emulated FP64 on the INT8 tensor cores (ozaki.cuh)
  int cdense_ctas = 0;   // CTAs per SM of k_condense_dense (runs beside the pair chain); 0: one CTA per tile
  int cdense_serial = 0; // 1: k_condense_dense on the caller's stream (no fork)
  int cdense_tma = 0;    // 1: the TMA-ring copy of the dense tiles (k_condense_dense_tma) instead of register staging
  int cond_prio = 1;     // 1: the pair chain at the highest launch priority, the dense tiles at the lowest
  int fac_prio = 0;      // 1: the factorization's panel kernels at the highest launch priority
  int cond_group = 8;    // batched pair tiles: scenarios per group of the (scenario group, tile, scenario) order
};
extern MdsVariant g_mds_var;

// true exactly once per (current device, key): guards per-device one-time setup
// such as cudaFuncSetAttribute (thread-safe; attributes are per device)
bool mds_once_per_device(const void* key);

template <typename... KArgs, typename... Args>
static inline cudaError_t launch_pdl(void (*k)(KArgs...), dim3 g, dim3 b, size_t smem, cudaStream_t st, Args... args) {
  const bool off = g_mds_var.no_pdl != 0;
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

// launch_pdl with an explicit scheduling priority (cudaLaunchAttributePriority; kept
// in captured graphs as the kernel node's priority).  prio = INT_MIN: none.
template <typename... KArgs, typename... Args>
static inline cudaError_t launch_pdl_prio(void (*k)(KArgs...), dim3 g, dim3 b, size_t smem, cudaStream_t st, int prio,
                                          Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = g;
  cfg.blockDim = b;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  int na = 0;
  if (!g_mds_var.no_pdl) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    na++;
  }
  if (prio != INT_MIN) {
    at[na].id = cudaLaunchAttributePriority;
    at[na].val.priority = prio;
    na++;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

// Cooperative + programmatic-dependent launch: for kernels whose CTAs meet at
// a software grid barrier (k_panel_exact).  The cooperative attribute makes
// the runtime guarantee that every CTA of the grid is resident at once (so
// the barrier cannot deadlock even when other streams' kernels share the GPU);
// the grid must not exceed the co-resident capacity (checked by the runtime).
template <typename... KArgs, typename... Args>
static inline cudaError_t launch_coop_pdl(void (*k)(KArgs...), dim3 g, dim3 b, size_t smem, cudaStream_t st,
                                          Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = g;
  cfg.blockDim = b;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[3];
  int na = 0;
  at[na].id = cudaLaunchAttributeCooperative;
  at[na].val.cooperative = 1;
  na++;
  if (!g_mds_var.no_pdl) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    na++;
  }
  if (g_mds_var.fac_prio) {   // (the panel chain ahead of the concurrent trailing update)
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    at[na].id = cudaLaunchAttributePriority;
    at[na].val.priority = hi;
    na++;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}
// the panel chain's launches: highest priority under variant fac_prio
static inline int chain_prio() {
  if (!g_mds_var.fac_prio) return INT_MIN;
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  return hi;
}

// ---------------------------------------------------------------------------
// launch accounting + optional per-class CUDA-event profiling (prof.cu)
enum MdsProfClass {
  PC_CONDENSE_W = 0, PC_CONDENSE_DENSE, PC_CONDENSE_YY, PC_ANORM, PC_PANEL_DIAG, PC_PANEL_TRSM,
  PC_PANEL_STORE, PC_PANEL_SLOW, PC_UPDATE, PC_FINALIZE, PC_SOLVE_GATHER, PC_SOLVE_FWD, PC_SOLVE_D,
  PC_SOLVE_BWD, PC_SOLVE_SCATTER, PC_RECOVER, PC_VECTORS, PC_CONDENSE_DIAG, PC_CONDENSE_COPY, PC_COUNT
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
