// Standalone timing harness for the panel kernels (not part of the library).
#define MDS_F1_TIMING 1
#include "../paper_2605_13736_b200/csrc/factor.cu"
#include "../paper_2605_13736_b200/csrc/prof.cu"
#include <cstdio>
#include <vector>
#include <random>
// a DMMA-saturating background load on every SM but one (smem-heavy so F1 cannot share an SM with it)
__global__ void k_busy(double* out, long long cycles, int mem) {
  extern __shared__ double bsm[];
  double a = threadIdx.x * 1e-3, b = 1.0 + blockIdx.x * 1e-6, c0 = 0.0, c1 = 0.0;
  const long long t0 = clock64();
  double* buf = out + 1024 + (size_t)blockIdx.x * (1 << 20);
  int it = 0;
  while (clock64() - t0 < cycles) {
#pragma unroll
    for (int k = 0; k < 64; k++) dmma(c0, c1, a, b);
    if (mem) { buf[(it * 256 + threadIdx.x) & ((1 << 20) - 1)] = c0; it++; }
  }
  bsm[threadIdx.x] = c0 + c1;
  if (c0 == 12345.0) out[blockIdx.x] = bsm[threadIdx.x ^ 1];
}
int main() {
  const int64_t N = 8192, ld = 8192;
  std::vector<double> h(N * ld);
  std::mt19937_64 rng(1);
  std::normal_distribution<double> nd;
  for (int64_t j = 0; j < N; j++) for (int64_t i = 0; i < N; i++) h[i + j * ld] = (i == j) ? 10.0 + nd(rng) : 0.01 * nd(rng);
  double* A; cudaMalloc(&A, sizeof(double) * N * ld);
  cudaMemcpy(A, h.data(), sizeof(double) * N * ld, cudaMemcpyHostToDevice);
  size_t wb = mds_factor_workspace_size(N);
  void* work; cudaMalloc(&work, wb); cudaMemset(work, 0, wb);
  FWork f = carve(work, N, nullptr);
  cudaFuncSetAttribute(k_panel_diag, cudaFuncAttributeMaxDynamicSharedMemorySize, F1SMEM);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int2 pi0 = make_int2(0, 64);
  cudaMemcpy(f.pinfo, &pi0, sizeof(int2), cudaMemcpyHostToDevice);
  for (int fuse = 0; fuse < 2; fuse++) {
    FWork fp = f;
    fp.fuse = fuse;
    fp.pidx = fuse;   // panel 1 (k0 = 64) with the deferred update of panel 0, or panel 0
    for (int it = 0; it < 3; it++) {
      cudaMemset(f.ctl, 0, sizeof(FCtl));
      k_panel_diag<<<1, 256, F1SMEM>>>(N, A, ld, fp);
    }
    cudaDeviceSynchronize();
    const int R = 200;
    cudaEventRecord(e0);
    for (int it = 0; it < R; it++) {
      k_panel_diag<<<1, 256, F1SMEM>>>(N, A, ld, fp);
    }
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long t[8]; cudaMemcpyFromSymbol(t, g_f1t, sizeof(t));
    printf("fuse=%d block0 panel %lld trailing %lld diaginv %lld\n", fuse, t[6]-t[1], t[5]-t[6], t[7]-t[2]);
    printf("fuse=%d k_panel_diag : %.2f us/launch (incl memset); phases (cycles): load+defer %lld fact %lld inv %lld out %lld total %lld  err=%s\n",
           fuse, ms * 1e3 / R, t[1] - t[0], t[2] - t[1], t[3] - t[2], t[4] - t[3], t[4] - t[0], cudaGetErrorString(cudaGetLastError()));
  }
  {
    cudaFuncSetAttribute(k_busy, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    double* junk; cudaMalloc(&junk, sizeof(double) * (1024 + 148ull * (1 << 20)));
    cudaStream_t s1, s2; cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking); cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
    FWork fp = f; fp.fuse = 1; fp.pidx = 1;
    for (int mem = 0; mem < 2; mem++) {
      k_busy<<<147, 256, 200 * 1024, s2>>>(junk, 40000000LL, mem);   // ~20 ms
      cudaEventRecord(e0, s1);
      for (int it = 0; it < 200; it++) k_panel_diag<<<1, 256, F1SMEM, s1>>>(N, A, ld, fp);
      cudaEventRecord(e1, s1);
      cudaDeviceSynchronize();
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      long long t[8]; cudaMemcpyFromSymbol(t, g_f1t, sizeof(t));
      printf("under DMMA load (mem=%d): %.2f us/launch; phases: load+defer %lld fact %lld inv %lld out %lld total %lld err=%s\n", mem,
             ms * 1e3 / 200, t[1] - t[0], t[2] - t[1], t[3] - t[2], t[4] - t[3], t[4] - t[0], cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
