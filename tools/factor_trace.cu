// Per-panel trace of k_panel_diag inside a full look-ahead factorization
// (wall time from %globaltimer, SM cycles from clock64).  Not part of the library.
#define MDS_F1_TRACE 1
#include "../paper_2605_13736_b200/csrc/factor.cu"
#include "../paper_2605_13736_b200/csrc/prof.cu"
#include <cstdio>
#include <random>
#include <vector>
#include <algorithm>
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
  const bool graph = argc > 2 && atoi(argv[2]) == 1;
  for (int i = 3; i + 1 < argc; i += 2) mds_set_variant(argv[i], atoll(argv[i + 1]));   // variant key value ...
  static unsigned long long uinit[4096][6];
  for (int i = 0; i < 4096; i++) { uinit[i][0] = uinit[i][3] = ~0ull; for (int k : {1, 2, 4, 5}) uinit[i][k] = 0; }
  double* A0; cudaMalloc(&A0, sizeof(double) * N * ld);
  cudaMemcpy(A0, h.data(), sizeof(double) * N * ld, cudaMemcpyHostToDevice);
  cudaGraphExec_t gexec = nullptr;
  if (graph) {
    cudaGraph_t g;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
    cudaMemcpyAsync(A, A0, sizeof(double) * N * ld, cudaMemcpyDeviceToDevice, st);
    int rc = mds_factor(N, A, ld, piv, -1.0, nullptr, ine, nullptr, status, work, wb, st);
    cudaStreamEndCapture(st, &g);
    cudaGraphInstantiate(&gexec, g, 0);
    if (rc) printf("capture rc %d\n", rc);
  }
  static unsigned long long usinit[512][160][2];
  for (int i = 0; i < 512; i++) for (int j = 0; j < 160; j++) { usinit[i][j][0] = ~0ull; usinit[i][j][1] = 0; }
  for (int rep = 0; rep < 3; rep++) {
    cudaMemcpyToSymbol(g_utrace, uinit, sizeof(uinit));
    cudaMemcpyToSymbol(g_usm, usinit, sizeof(usinit));
    static unsigned long long f4init[4096][2];
    for (int i = 0; i < 4096; i++) { f4init[i][0] = ~0ull; f4init[i][1] = 0; }
    cudaMemcpyToSymbol(g_f4trace, f4init, sizeof(f4init));
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    if (graph) {
      cudaEventRecord(a, st); cudaGraphLaunch(gexec, st); cudaEventRecord(b, st);
    } else {
      cudaMemcpyAsync(A, A0, sizeof(double) * N * ld, cudaMemcpyDeviceToDevice, st);
      cudaEventRecord(a, st);
      int rc = mds_factor(N, A, ld, piv, -1.0, nullptr, ine, nullptr, status, work, wb, st);
      cudaEventRecord(b, st);
      if (rc) printf("rc %d\n", rc);
    }
    cudaStreamSynchronize(st);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("rep %d (%s): %.3f ms\n", rep, graph ? "graph" : "eager", ms);
  }
  static unsigned long long ut[4096][6];
  cudaMemcpyFromSymbol(ut, g_utrace, sizeof(ut));
  static unsigned long long usm[512][160][2];
  cudaMemcpyFromSymbol(usm, g_usm, sizeof(usm));
  static unsigned f1sm[4096];
  cudaMemcpyFromSymbol(f1sm, g_f1sm, sizeof(f1sm));
  static unsigned long long tr[4096][8];
  cudaMemcpyFromSymbol(tr, g_f1trace, sizeof(tr));
  const int np = (int)((N + 62) / 63) + 1;
  unsigned long long t0 = tr[0][0];
  double sum_us = 0, sum_cyc = 0;
  int n = 0;
  for (int p = 0; p < np; p++) {
    if (!tr[p][0] || !tr[p][6]) continue;
    const double us = (tr[p][6] - tr[p][0]) * 1e-3, cyc = (double)(tr[p][7] - tr[p][1]);
    if (p < 12 || p % 8 == 0) {
      auto ab = [&](unsigned long long t) { return (t == ~0ull || t == 0) ? -1.0 : ((double)t - (double)t0) * 1e-3; };
      printf("  abs: F1 [%.1f, %.1f] on SM %u  trsm [%.1f, %.1f]  U [%.1f, %.1f]", ab(tr[p][0]), ab(tr[p][6]), f1sm[p], ab(ut[p][3]), ab(ut[p][4]), ab(ut[p][0]), ab(ut[p][1]));
      if (p > 0 && p < 512) {
        int nsm = 0; double late = 0;
        for (int k = 0; k < 160; k++) if (usm[p - 1][k][0] != ~0ull) { nsm++; late = std::max(late, ab(usm[p - 1][k][0])); }
        const unsigned sm = f1sm[p];
        printf(" | U(p-1): %d SMs, last CTA start %.1f; U(p-1) on F1's SM: [%.1f, %.1f]", nsm, late, ab(usm[p - 1][sm][0]), ab(usm[p - 1][sm][1]));
      }
      printf("\n");
      auto rel = [&](unsigned long long t) { return (t == ~0ull || t == 0) ? -1.0 : ((double)t - (double)tr[p][0]) * 1e-3; };
      printf("panel %3d start %8.1f us  F1 %5.1f us (%.0f MHz; defer %llu fact %llu inv %llu cyc) | U(p) [%.1f, %.1f] F2-in-U(p) %llu | trsm [%.1f, %.1f] tiles %llu\n", p,
             (tr[p][0] - t0) * 1e-3, us, cyc / us, tr[p][3] - tr[p][1], tr[p][5] - tr[p][3], tr[p][7] - tr[p][5],
             rel(ut[p][0]), rel(ut[p][1]), p > 0 ? ut[p - 1][2] : 0ull, rel(ut[p][3]), rel(ut[p][4]), ut[p][5]);
    }
    sum_us += us; sum_cyc += cyc; n++;
  }
  printf("avg F1 %.1f us %.0f cycles over %d panels; err=%s\n", sum_us / n, sum_cyc / n, n, cudaGetErrorString(cudaGetLastError()));
  // per panel (absolute us from the first F1): F1 start/end, trsm start/end, U start/end, gap U(p-1) end -> U(p) start
  static unsigned long long f4[4096][2];
  cudaMemcpyFromSymbol(f4, g_f4trace, sizeof(f4));
  printf("csv,p,f1s,f1e,trs,tre,us,ue,gap,f4s,f4e\n");
  double prev_ue = -1;
  for (int p = 0; p < np; p++) {
    if (!tr[p][0]) continue;
    auto ab = [&](unsigned long long t) { return (t == ~0ull || t == 0) ? -1.0 : ((double)t - (double)t0) * 1e-3; };
    const double us = ab(ut[p][0]), ue = ab(ut[p][1]);
    printf("csv,%d,%.2f,%.2f,%.2f,%.2f,%.2f,%.2f,%.2f,%.2f,%.2f\n", p, ab(tr[p][0]), ab(tr[p][6]), ab(ut[p][3]), ab(ut[p][4]), us, ue,
           (prev_ue >= 0 && us >= 0) ? us - prev_ue : -1.0, ab(f4[p][0]), ab(f4[p][1]));
    prev_ue = ue;
  }
  return 0;
}
