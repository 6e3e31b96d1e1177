// Standalone timing harness for the panel kernels (not part of the library).
#define MDS_F1_TIMING 1
#include "../paper_2605_13736_b200/csrc/factor.cu"
#include "../paper_2605_13736_b200/csrc/prof.cu"
#include <cstdio>
#include <vector>
#include <random>
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
  for (int it = 0; it < 3; it++) {
    cudaMemset(f.ctl, 0, sizeof(FCtl));
    k_panel_diag<<<1, 256, F1SMEM>>>(N, A, ld, f);
  }
  cudaDeviceSynchronize();
  const int R = 200;
  cudaEventRecord(e0);
  for (int it = 0; it < R; it++) {
    cudaMemsetAsync(f.ctl, 0, 16);
    k_panel_diag<<<1, 256, F1SMEM>>>(N, A, ld, f);
  }
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long t[8]; cudaMemcpyFromSymbol(t, g_f1t, sizeof(t));
  printf("block0 panel %lld trailing %lld diaginv %lld\n", t[6]-t[1], t[5]-t[6], t[7]-t[2]);
  printf("k_panel_diag: %.2f us/launch (incl memset); phases (cycles): load %lld fact %lld inv %lld out %lld total %lld  err=%s\n",
         ms * 1e3 / R, t[1] - t[0], t[2] - t[1], t[3] - t[2], t[4] - t[3], t[4] - t[0], cudaGetErrorString(cudaGetLastError()));
  return 0;
}
