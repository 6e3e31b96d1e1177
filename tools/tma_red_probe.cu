// probe: does TMA reduce-add (cp.reduce.async.bulk.tensor .add) work on FP64 tensor maps?
#include <cuda.h>
#include <cstdio>
#include <vector>
typedef CUresult (*PFN)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
__global__ void k(const __grid_constant__ CUtensorMap m) {
  __shared__ alignas(1024) double buf[8 * 64];
  for (int i = threadIdx.x; i < 512; i += blockDim.x) buf[i] = 0.5 + i;   // [col][8 rows]
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned s = (unsigned)__cvta_generic_to_shared(buf);
    asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%1, %2}], [%3];" :: "l"(&m), "r"(8), "r"(0), "r"(s) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}
int main() {
  const int R = 64, C = 64;
  std::vector<double> h(R * C);
  for (int i = 0; i < R * C; i++) h[i] = 1000.0 * i;
  double* d; cudaMalloc(&d, sizeof(double) * R * C);
  cudaMemcpy(d, h.data(), sizeof(double) * R * C, cudaMemcpyHostToDevice);
  void* fn; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  CUtensorMap m;
  cuuint64_t dims[2] = {R, C}, str[1] = {R * 8};
  cuuint32_t box[2] = {8, 64}, es[2] = {1, 1};
  CUresult r = ((PFN)fn)(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  k<<<1, 128>>>(m);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<double> o(R * C);
  cudaMemcpy(o.data(), d, sizeof(double) * R * C, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int c = 0; c < C; c++)
    for (int rr = 0; rr < R; rr++) {
      double exp = h[rr + c * R] + ((rr >= 8 && rr < 16) ? (0.5 + (c * 8 + (rr - 8))) : 0.0);
      if (o[rr + c * R] != exp) bad++;
    }
  printf("encode=%d launch=%s mismatches=%d sample %.1f (exp %.1f)\n", (int)r, cudaGetErrorString(e), bad, o[8], h[8] + 0.5);
}
