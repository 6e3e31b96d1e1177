// probe: per-SM TMA load throughput for the trailing-update operand tiles
// (64 rows x 64 k FP64 = 32 KB per operand, 2 operands per tile) as a function
// of the box shape / swizzle / storage layout.  148 CTAs, producer lane issues
// loads into a 3-stage mbarrier ring, a consumer lane just waits and releases.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_bw_probe tools/tma_bw_probe.cu -lcuda
#include <cuda.h>
#include <cstdio>
#include <vector>
typedef CUresult (*PFN)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
constexpr int STAGES = 3, STAGEB = 65536;

__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
  asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n" ::"r"(bar),
               "r"(parity) : "memory");
}
// mode 0: column-major, box {b0 rows, 64 k}: 64/b0 boxes per operand, coords (row, k)
// mode 1: row-major (k contiguous), box {b0 k, 64 rows}: 64/b0 boxes per operand, coords (k, row)
__global__ void __launch_bounds__(64) kprobe(const __grid_constant__ CUtensorMap mL, const __grid_constant__ CUtensorMap mW,
                                            int mode, int b0, int tiles, int nrows, unsigned long long* cyc) {
  extern __shared__ unsigned char raw[];
  const unsigned base = ((unsigned)__cvta_generic_to_shared(raw) + 1023u) & ~1023u;
  const unsigned full0 = base + STAGES * STAGEB, empty0 = full0 + 8 * STAGES;
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; i++) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(full0 + 8 * i));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(empty0 + 8 * i));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const long long t0 = clock64();
  const int nb = 64 / b0, boxb = 32768 / nb;
  if (threadIdx.x == 0) {
    for (int i = 0; i < tiles; i++) {
      const int st = i % STAGES, u = i / STAGES;
      if (u > 0) mbar_wait(empty0 + 8 * st, (u - 1) & 1);
      const unsigned fb = full0 + 8 * st, sL = base + st * STAGEB, sW = sL + 32768;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb), "r"(STAGEB) : "memory");
      const int r0 = (int)(((long long)(blockIdx.x * 7919 + i * 131) * 64) % nrows);
      const int c0 = (int)(((long long)(blockIdx.x * 104729 + i * 37) * 64) % nrows);
      for (int b = 0; b < nb; b++) {
        int x0, y0, x1, y1;
        if (mode == 0) { x0 = r0 + b * b0; y0 = 0; x1 = c0 + b * b0; y1 = 0; }
        else { x0 = b * b0; y0 = r0; x1 = b * b0; y1 = c0; }
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                         sL + b * boxb), "l"(&mL), "r"(x0), "r"(y0), "r"(fb) : "memory");
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                         sW + b * boxb), "l"(&mW), "r"(x1), "r"(y1), "r"(fb) : "memory");
      }
    }
  } else if (threadIdx.x == 32) {
    for (int i = 0; i < tiles; i++) {
      const int st = i % STAGES, u = i / STAGES;
      mbar_wait(full0 + 8 * st, u & 1);
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(empty0 + 8 * st) : "memory");
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}

int main() {
  const int nrows = 8192;
  double *L, *W;
  cudaMalloc(&L, sizeof(double) * nrows * 64);
  cudaMalloc(&W, sizeof(double) * nrows * 64);
  cudaMemset(L, 0, sizeof(double) * nrows * 64);
  cudaMemset(W, 0, sizeof(double) * nrows * 64);
  unsigned long long* cyc;
  cudaMalloc(&cyc, 8 * 148);
  void* fn;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  cudaFuncSetAttribute(kprobe, cudaFuncAttributeMaxDynamicSharedMemorySize, STAGES * STAGEB + 2048);
  struct V { int mode, b0; CUtensorMapSwizzle sw; const char* name; };
  V vs[] = {{0, 8, CU_TENSOR_MAP_SWIZZLE_64B, "colmajor box{8 rows,64k} sw64 (current)"},
            {0, 16, CU_TENSOR_MAP_SWIZZLE_128B, "colmajor box{16 rows,64k} sw128"},
            {0, 32, CU_TENSOR_MAP_SWIZZLE_NONE, "colmajor box{32 rows,64k} none"},
            {0, 64, CU_TENSOR_MAP_SWIZZLE_NONE, "colmajor box{64 rows,64k} none"},
            {1, 8, CU_TENSOR_MAP_SWIZZLE_64B, "rowmajor box{8 k,64 rows} sw64"},
            {1, 16, CU_TENSOR_MAP_SWIZZLE_128B, "rowmajor box{16 k,64 rows} sw128"},
            {1, 64, CU_TENSOR_MAP_SWIZZLE_NONE, "rowmajor box{64 k,64 rows} none"}};
  for (const V& v : vs) {
    CUtensorMap m[2];
    double* bufs[2] = {L, W};
    bool ok = true;
    for (int j = 0; j < 2; j++) {
      cuuint64_t dims[2], str[1];
      cuuint32_t box[2], es[2] = {1, 1};
      if (v.mode == 0) { dims[0] = nrows; dims[1] = 64; str[0] = nrows * 8; box[0] = v.b0; box[1] = 64; }
      else { dims[0] = 64; dims[1] = nrows; str[0] = 64 * 8; box[0] = v.b0; box[1] = 64; }
      CUresult r = ((PFN)fn)(&m[j], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, bufs[j], dims, str, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, v.sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) { printf("%s: encode failed %d\n", v.name, (int)r); ok = false; }
    }
    if (!ok) continue;
    const int tiles = 2000;
    kprobe<<<148, 64, STAGES * STAGEB + 2048>>>(m[0], m[1], v.mode, v.b0, 50, nrows, cyc);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    kprobe<<<148, 64, STAGES * STAGEB + 2048>>>(m[0], m[1], v.mode, v.b0, tiles, nrows, cyc);
    cudaEventRecord(b);
    cudaError_t e = cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    std::vector<unsigned long long> h(148);
    cudaMemcpy(h.data(), cyc, 8 * 148, cudaMemcpyDeviceToHost);
    double mean = 0; for (auto c : h) mean += c; mean /= 148;
    const double bytes = 148.0 * tiles * STAGEB;
    printf("{\"variant\": \"%s\", \"err\": \"%s\", \"ms\": %.3f, \"TB_s\": %.2f, \"B_per_clk_per_SM\": %.1f}\n", v.name,
           cudaGetErrorString(e), ms, bytes / (ms * 1e-3) / 1e12, (double)tiles * STAGEB / mean);
  }
}
