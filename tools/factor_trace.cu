// Per-panel trace of k_panel_diag inside a full look-ahead factorization
// (wall time from %globaltimer, SM cycles from clock64).  Not part of the library.
#define MDS_F1_TRACE 1
#include "../paper_2605_13736_b200/csrc/factor.cu"
#include "../paper_2605_13736_b200/csrc/prof.cu"
#include <cstdio>
#include <random>
#include <vector>
int main(int argc, char** argv) {
  const int64_t N = argc > 1 ? atoll(argv[1]) : 8192, ld = N;
  std::vector<double> h(N * ld);
  std::mt19937_64 rng(1);
  std::normal_distribution<double> nd;
  // quasi-definite: [[D+, B^T],[B, -D-]] with small off-diagonal coupling
  for (int64_t j = 0; j < N; j++)
    for (int64_t i = j; i < N; i++) h[i + j * ld] = (i == j) ? ((j < N / 2) ? 4.0 : -4.0) + 0.1 * nd(rng) : 0.02 * nd(rng);
  double* A; cudaMalloc(&A, sizeof(double) * N * ld);
  size_t wb = mds_factor_workspace_size(N);
  void* work; cudaMalloc(&work, wb);
  int32_t* piv; cudaMalloc(&piv, sizeof(int32_t) * 2 * N);
  mds_inertia* ine; cudaMalloc(&ine, sizeof(mds_inertia));
  int32_t* status; cudaMalloc(&status, 4);
  cudaStream_t st; cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  for (int rep = 0; rep < 2; rep++) {
    cudaMemcpy(A, h.data(), sizeof(double) * N * ld, cudaMemcpyHostToDevice);
    cudaMemset(status, 0, 4);
    int rc = mds_factor(N, A, ld, piv, -1.0, ine, nullptr, status, work, wb, st);
    cudaStreamSynchronize(st);
    if (rc) printf("rc %d\n", rc);
  }
  static unsigned long long tr[4096][8];
  cudaMemcpyFromSymbol(tr, g_f1trace, sizeof(tr));
  const int np = (int)((N + 62) / 63) + 1;
  unsigned long long t0 = tr[0][0];
  double sum_us = 0, sum_cyc = 0;
  int n = 0;
  for (int p = 0; p < np; p++) {
    if (!tr[p][0] || !tr[p][6]) continue;
    const double us = (tr[p][6] - tr[p][0]) * 1e-3, cyc = (double)(tr[p][7] - tr[p][1]);
    if (p % 8 == 0)
      printf("panel %3d start %8.1f us  F1 %6.1f us  %7.0f cycles (%.0f MHz): load+defer %llu fact %llu inv+out %llu\n", p,
             (tr[p][0] - t0) * 1e-3, us, cyc, cyc / us, tr[p][3] - tr[p][1], tr[p][5] - tr[p][3], tr[p][7] - tr[p][5]);
    sum_us += us; sum_cyc += cyc; n++;
  }
  printf("avg F1 %.1f us %.0f cycles over %d panels; err=%s\n", sum_us / n, sum_cyc / n, n, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
