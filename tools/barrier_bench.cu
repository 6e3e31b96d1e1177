// Grid-barrier latency probe: G CTAs x 512 threads, R barriers of the k_panel_exact kind
// (bar.sync; thread 0: red.release.gpu + acquire spin; bar.sync; partial reads), vs a
// thread-block-cluster barrier (barrier.cluster) with DSMEM partials.  Not part of the library.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
  unsigned v; asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v;
}
__global__ void __launch_bounds__(512) k_grid(unsigned* ctr, double* part, int R, double* out) {
  __shared__ double sh[32];
  double acc = 0.0;
  for (int it = 0; it < R; it++) {
    double* bank = part + 512 * (it & 1);
    if (threadIdx.x == 0) bank[blockIdx.x] = it + blockIdx.x;
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
      const unsigned target = (unsigned)(it + 1) * gridDim.x;
      while (ld_acq(ctr) < target) {}
    }
    __syncthreads();
    double a = -1.0;
    for (int c = threadIdx.x; c < (int)gridDim.x; c += blockDim.x) a = fmax(a, __ldcg(&bank[c]));
    for (int o = 16; o; o >>= 1) a = fmax(a, __shfl_xor_sync(0xffffffffu, a, o));
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = a;
    __syncthreads();
    if (threadIdx.x < 32) { a = (threadIdx.x < 16) ? sh[threadIdx.x] : -1.0; for (int o = 16; o; o >>= 1) a = fmax(a, __shfl_xor_sync(0xffffffffu, a, o)); if (threadIdx.x == 0) sh[31] = a; }
    __syncthreads();
    acc += sh[31];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = acc;
}
__global__ void __launch_bounds__(512) k_cluster(int R, double* out) {
  cg::cluster_group cl = cg::this_cluster();
  __shared__ double part[2][16];
  __shared__ double sh[32];
  double acc = 0.0;
  const unsigned rank = cl.block_rank(), n = cl.num_blocks();
  for (int it = 0; it < R; it++) {
    if (threadIdx.x == 0) {
      double* dst = cl.map_shared_rank(&part[it & 1][0], 0);
      dst[rank] = it + rank;
    }
    cl.sync();
    double a = -1.0;
    if (threadIdx.x < n) a = *cl.map_shared_rank(&part[it & 1][threadIdx.x], 0);
    for (int o = 16; o; o >>= 1) a = fmax(a, __shfl_xor_sync(0xffffffffu, a, o));
    if (threadIdx.x == 0) sh[31] = a;
    __syncthreads();
    acc += sh[31];
  }
  cl.sync();
  if (threadIdx.x == 0) out[blockIdx.x] = acc;
}
int main() {
  unsigned* ctr; double *part, *out;
  cudaMalloc(&ctr, 4); cudaMalloc(&part, 1024 * 8); cudaMalloc(&out, 4096 * 8);
  const int R = 2000;
  for (int G : {8, 16, 32, 64, 128}) {
    cudaMemset(ctr, 0, 4);
    void* args[] = {&ctr, &part, (void*)&R, &out};
    int Rv = R; args[2] = &Rv;
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void*)k_grid, G, 512, args, 0, 0);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("grid barrier G=%3d: %.3f us per barrier (%s)\n", G, ms * 1e3 / R, cudaGetErrorString(cudaGetLastError()));
  }
  for (int C : {8, 16}) {
    cudaFuncSetAttribute(k_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(C); cfg.blockDim = dim3(512);
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    cudaError_t e = cudaLaunchKernelEx(&cfg, k_cluster, R, out);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("cluster barrier C=%2d: %.3f us per barrier (%s / %s)\n", C, ms * 1e3 / R, cudaGetErrorString(e), cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
