// Per-phase cycles of the multi-CTA exact Bunch-Kaufman panel (CTA 0, summed over every
// exact column) on a pivot-heavy symmetric matrix (zero diagonal: no 1x1 pivot passes the
// speculative test).  Not part of the library.  usage: exact_trace [N]
#define MDS_F1_TRACE 1
#include "../paper_2605_13736_b200/csrc/factor.cu"
#include "../paper_2605_13736_b200/csrc/prof.cu"
#include <cstdio>
#include <random>
#include <vector>
int main(int argc, char** argv) {
  const int64_t N = argc > 1 ? atoll(argv[1]) : 8192, ld = N;
  std::vector<double> h(N * ld);
  std::mt19937_64 rng(3);
  std::normal_distribution<double> nd;
  for (int64_t j = 0; j < N; j++)
    for (int64_t i = j; i < N; i++) h[i + j * ld] = (i == j) ? 0.05 * nd(rng) : nd(rng) / sqrt((double)N);
  double *A, *A0;
  cudaMalloc(&A, sizeof(double) * N * ld);
  cudaMalloc(&A0, sizeof(double) * N * ld);
  cudaMemcpy(A0, h.data(), sizeof(double) * N * ld, cudaMemcpyHostToDevice);
  size_t wb = mds_factor_workspace_size(N);
  void* work; cudaMalloc(&work, wb);
  int32_t* piv; cudaMalloc(&piv, sizeof(int32_t) * 2 * N);
  mds_inertia* ine; cudaMalloc(&ine, sizeof(mds_inertia));
  int32_t* status; cudaMalloc(&status, 4);
  cudaStream_t st; cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  for (int rep = 0; rep < 2; rep++) {
    unsigned long long z[10] = {0};
    cudaMemcpyToSymbol(g_xph, z, sizeof(z));
    cudaMemcpyAsync(A, A0, sizeof(double) * N * ld, cudaMemcpyDeviceToDevice, st);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a, st);
    int rc = mds_factor(N, A, ld, piv, -1.0, nullptr, ine, nullptr, status, work, wb, st);
    cudaEventRecord(b, st);
    cudaStreamSynchronize(st);
    float ms; cudaEventElapsedTime(&ms, a, b);
    unsigned long long ph[10];
    cudaMemcpyFromSymbol(ph, g_xph, sizeof(ph));
    FCtl c; cudaMemcpy(&c, work, sizeof(FCtl), cudaMemcpyDeviceToHost);
    printf("rep %d rc %d: factor %.2f ms, exact columns %d, swaps %d, iterations %llu\n", rep, rc, ms, c.nexact, c.nswap, ph[9]);
    const char* nm[8] = {"wrow", "gemv", "cta_argmax", "exchange", "candidate", "interchange", "scaling", "end_sync"};
    double tot = 0; for (int i = 0; i < 8; i++) tot += ph[i];
    for (int i = 0; i < 8; i++)
      printf("  %-12s %10.0f cycles/iter  %5.1f %%\n", nm[i], ph[9] ? (double)ph[i] / ph[9] : 0.0, 100.0 * ph[i] / tot);
    printf("  total %.0f cycles/iter = %.2f us/iter at 1.965 GHz\n", tot / ph[9], tot / ph[9] / 1965.0);
  }
  return 0;
}
