// dist.cu — device kernels of the distributed Bunch-Kaufman LDL^T of ONE
// system across GPUs (the paper's method is single-GPU,
// "does not support distributed memory parallelism", and
// leaves larger systems to future work).
//
// Layout (paper_2605_13736_b200/dist.py drives it): the lower triangle of M is
// cut into 64-column panels, panel g owned by rank g mod P (1-D block-cyclic),
// each rank storing its panels full height (column-major, ld = N).  Panel g:
//   owner:  mds_dist_panel   -- the speculative (unpivoted) LDL^T of the panel:
//                               F1 on the 64x64 diagonal block, F2 W21 = A21 L11^-T,
//                               L21 = W21 D^-1, and the Bunch-Kaufman 1x1 acceptance
//                               test |d_j| >= alpha colmax_j of every column
//                               (reading R3 of DESIGN.md);
//   all:    broadcast of (L, W) of the panel, then mds_dist_update on the
//           rank's own later panels: C -= L W^T (FP64 DMMA tiles).
// A panel that fails the test ends the distributed phase: the Schur complement
// (all panels from it on) is gathered on one rank and factored there by
// mds_factor (exact BK); inertia(M) = inertia(D_1) + inertia(S) (Haynsworth,
// PAPER.md:191).  The solve (mds_dist_trsv64, mds_dist_gemv_*) follows the same
// block form.  Product path only (not shared with oracle/).
#include "common.cuh"

namespace {
constexpr int DB = 64;                                                  // panel width
constexpr int DP = DB + 1;                                              // smem stride (banks)
constexpr double DALPHA = 0.64038820320220756872767623199676;           // (1 + sqrt(17)) / 8

__device__ __forceinline__ void dp_dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
__device__ __forceinline__ void atomic_max_nonneg(double* p, double v) {   // |x| values: IEEE order = int order
  atomicMax(reinterpret_cast<unsigned long long*>(p), (unsigned long long)__double_as_longlong(v));
}

// F1: the nb x nb diagonal block A (lower, column-major, lda), right-looking
// unpivoted LDL^T.  Outputs rows 0..nb-1 of the panel: L (unit lower), W(i, j) =
// the column j at its elimination (W(j, j) = d_j), d[j], cmax[j] = max_{j<i<nb} |W(i, j)|.
__global__ void __launch_bounds__(256) k_dp_f1(int nb, const double* __restrict__ A, int64_t lda, double* L,
                                               double* W, int64_t ldl, double* d, double* cmax) {
  __shared__ double S[DB * DP];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < DB * DB; e += blockDim.x) {
    const int i = e % DB, j = e / DB;
    S[j * DP + i] = (i < nb && j < nb && i >= j) ? A[i + (int64_t)j * lda] : 0.0;
  }
  __syncthreads();
  for (int j = 0; j < nb; j++) {
    const double dj = S[j * DP + j];
    const double rd = dj != 0.0 ? 1.0 / dj : 0.0;
    if (warp == 0) {
      double cm = 0.0;
      for (int i = j + 1 + lane; i < nb; i += 32) cm = fmax(cm, fabs(S[j * DP + i]));
      cm = warp_max(cm);
      if (lane == 0) { cmax[j] = cm; d[j] = dj; }
    }
    for (int i = j + tid; i < nb; i += blockDim.x) {
      const double wij = S[j * DP + i];
      W[i + (int64_t)j * ldl] = wij;
      L[i + (int64_t)j * ldl] = (i == j) ? 1.0 : wij * rd;
    }
    const int m = nb - j - 1;
    for (int e = tid; e < m * m; e += blockDim.x) {
      const int i = j + 1 + e % m, c = j + 1 + e / m;
      if (i >= c) S[c * DP + i] -= (S[j * DP + i] * rd) * S[j * DP + c];
    }
    __syncthreads();
  }
}

// F2: rows nb..n-1 of the panel.  Per row (one thread): W(i, j) = A(i, j) -
// sum_{t<j} W(i, t) L(j, t) (A21 = W21 L11^T), L(i, j) = W(i, j) / d_j; per-CTA
// column maxima of |W| into parts[blockIdx.x][j].
template <int NBC>
__global__ void __launch_bounds__(128) k_dp_f2(int64_t n, int nb, const double* __restrict__ A, int64_t lda, double* L,
                                               double* W, int64_t ldl, const double* __restrict__ d, double* parts) {
  __shared__ double L11[DB * DB];
  __shared__ double rdv[DB];
  __shared__ double cm[DB];
  const int tid = threadIdx.x;
  for (int e = tid; e < DB * DB; e += blockDim.x) {
    const int r = e % DB, c = e / DB;
    L11[r * DB + c] = (r < nb && c < nb && r > c) ? L[r + (int64_t)c * ldl] : 0.0;   // row-major L11(r, c)
  }
  if (tid < DB) {
    rdv[tid] = (tid < nb && d[tid] != 0.0) ? 1.0 / d[tid] : 0.0;
    cm[tid] = 0.0;
  }
  __syncthreads();
  const int64_t i = nb + (int64_t)blockIdx.x * blockDim.x + tid;
  double w[NBC];
  if (i < n) {
#pragma unroll
    for (int j = 0; j < NBC; j++) w[j] = (j < nb) ? A[i + (int64_t)j * lda] : 0.0;
#pragma unroll
    for (int j = 1; j < NBC; j++) {
      double s = w[j];
#pragma unroll
      for (int t = 0; t < j; t++) s = fma(-w[t], L11[j * DB + t], s);
      w[j] = s;
    }
#pragma unroll
    for (int j = 0; j < NBC; j++) {
      if (j < nb) {
        W[i + (int64_t)j * ldl] = w[j];
        L[i + (int64_t)j * ldl] = w[j] * rdv[j];
      }
    }
  } else {
#pragma unroll
    for (int j = 0; j < NBC; j++) w[j] = 0.0;
  }
#pragma unroll
  for (int j = 0; j < NBC; j++) {
    const double v = warp_max(fabs(w[j]));
    if ((tid & 31) == 0 && v > 0.0) atomic_max_nonneg(&cm[j], v);
  }
  __syncthreads();
  if (tid < DB) parts[(int64_t)blockIdx.x * DB + tid] = cm[tid];
}

// Acceptance (one CTA of 64 threads): colmax_j = max(in-block, F2 parts); the
// panel is accepted when every column passes |d_j| >= alpha colmax_j (the BK 1x1
// test without interchange; 0 >= 0 accepts an exactly zero column).  Then the
// inertia of D_1 (tol) is added to inertia[3] and accepted[0] = 1, else 0.
__global__ void __launch_bounds__(DB) k_dp_accept(int nb, const double* d, const double* cmax, const double* parts,
                                                  int nparts, double tol, int32_t* accepted, long long* inertia) {
  const int j = threadIdx.x;
  bool ok = true;
  double dj = 0.0;
  if (j < nb) {
    double cm = cmax[j];
    for (int t = 0; t < nparts; t++) cm = fmax(cm, parts[(int64_t)t * DB + j]);
    dj = d[j];
    ok = fabs(dj) >= DALPHA * cm;
  }
  const int all = __syncthreads_and(ok ? 1 : 0);
  const int pos = __syncthreads_count(j < nb && dj > tol);
  const int neg = __syncthreads_count(j < nb && dj < -tol);
  if (j == 0) {
    accepted[0] = all;
    if (all) {
      inertia[0] += pos;
      inertia[2] += neg;
      inertia[1] += nb - pos - neg;
    }
  }
}

// Trailing update of one rank's later panels: for local panel q (global first
// column kq[q], width wq[q], stored at C + q * DB * ldc, rows global), rows i >= kq:
// C(i, c) -= sum_t L(i - k0, t) W(c - k0, t).  One CTA per (64-row tile, panel);
// 8 warps x (32 x 16) of DMMA m8n8k4.
__global__ void __launch_bounds__(256) k_dp_update(int64_t N, int64_t k0, int nb, const double* __restrict__ L,
                                                   const double* __restrict__ W, int64_t ldl, double* C, int64_t ldc,
                                                   const int64_t* kq, const int* wq) {
  constexpr int KH = DB / 2;        // k in two halves (static shared memory)
  __shared__ double Ls[KH * DP];   // Ls[t * DP + r] = L(r0 + r, kh + t)
  __shared__ double Ws[KH * DP];   // Ws[t * DP + c] = W(kq + c, kh + t)
  const int q = blockIdx.y;
  const int64_t c0 = kq[q];
  const int w = wq[q];
  const int64_t r0 = c0 + (int64_t)blockIdx.x * DB;
  if (r0 >= N) return;
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31, g = lane >> 2, qq = lane & 3;
  const int wm = (warp & 1) * 32, wn = (warp >> 1) * 16;
  double acc[4][2][2];
#pragma unroll
  for (int a = 0; a < 4; a++)
#pragma unroll
    for (int b = 0; b < 2; b++) acc[a][b][0] = acc[a][b][1] = 0.0;
  for (int kh = 0; kh < nb; kh += KH) {
    __syncthreads();
    for (int e = tid; e < KH * DB; e += blockDim.x) {
      const int r = e % DB, t = kh + e / DB;
      const int64_t gi = r0 + r, gc = c0 + r;
      Ls[(t - kh) * DP + r] = (t < nb && gi < N) ? L[(gi - k0) + (int64_t)t * ldl] : 0.0;
      Ws[(t - kh) * DP + r] = (t < nb && r < w) ? W[(gc - k0) + (int64_t)t * ldl] : 0.0;
    }
    __syncthreads();
    const int kn = (nb - kh < KH ? nb - kh : KH);
    for (int t0 = 0; t0 < kn; t0 += 4) {
      double av[4], bv[2];
#pragma unroll
      for (int a = 0; a < 4; a++) av[a] = Ls[(t0 + qq) * DP + wm + 8 * a + g];
#pragma unroll
      for (int b = 0; b < 2; b++) bv[b] = Ws[(t0 + qq) * DP + wn + 8 * b + g];
#pragma unroll
      for (int a = 0; a < 4; a++)
#pragma unroll
        for (int b = 0; b < 2; b++) dp_dmma(acc[a][b][0], acc[a][b][1], av[a], bv[b]);
    }
  }
  double* Cq = C + (int64_t)q * DB * ldc;
#pragma unroll
  for (int a = 0; a < 4; a++)
#pragma unroll
    for (int b = 0; b < 2; b++)
#pragma unroll
      for (int e = 0; e < 2; e++) {
        const int r = wm + 8 * a + g, c = wn + 8 * b + 2 * qq + e;
        const int64_t gi = r0 + r;
        if (gi < N && c < w && gi >= c0 + c) Cq[gi + (int64_t)c * ldc] -= acc[a][b][e];
      }
}

// 64 x 64 unit-lower triangular solve with one vector (one CTA of 64 threads):
// mode 0: y := L11^-1 y; mode 1: y := L11^-T y.  L11 = rows / columns 0..nb-1 at L (ldl).
__global__ void __launch_bounds__(DB) k_dp_trsv64(int nb, const double* __restrict__ L, int64_t ldl, double* y,
                                                  int mode) {
  __shared__ double ys[DB];
  const int i = threadIdx.x;
  ys[i] = i < nb ? y[i] : 0.0;
  __syncthreads();
  if (mode == 0) {
    for (int j = 0; j < nb; j++) {
      const double yj = ys[j];
      __syncthreads();
      if (i > j && i < nb) ys[i] = fma(-L[i + (int64_t)j * ldl], yj, ys[i]);
      __syncthreads();
    }
  } else {
    for (int j = nb - 1; j >= 0; j--) {
      const double yj = ys[j];
      __syncthreads();
      if (i < j) ys[i] = fma(-L[j + (int64_t)i * ldl], yj, ys[i]);
      __syncthreads();
    }
  }
  if (i < nb) y[i] = ys[i];
}

// acc[i] += sum_{t<nb} L(i, t) y[t] for rows i in [r0, r1) of the panel block (one thread per row)
__global__ void __launch_bounds__(256) k_dp_gemv_n(int64_t r0, int64_t r1, int nb, const double* __restrict__ L,
                                                   int64_t ldl, const double* __restrict__ y, double* acc) {
  const int64_t i = r0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= r1) return;
  double s = 0.0;
  for (int t = 0; t < nb; t++) s = fma(L[i + (int64_t)t * ldl], y[t], s);
  acc[i] += s;
}

// out[t] = sum_{i in [r0, r1)} L(i, t) x[i] for t < nb (one CTA per column, fixed-order tree)
__global__ void __launch_bounds__(256) k_dp_gemv_t(int64_t r0, int64_t r1, const double* __restrict__ L, int64_t ldl,
                                                   const double* __restrict__ x, double* out) {
  __shared__ double red[8];
  const int t = blockIdx.x, tid = threadIdx.x;
  double s = 0.0;
  for (int64_t i = r0 + tid; i < r1; i += blockDim.x) s = fma(L[i + (int64_t)t * ldl], x[i], s);
  s = warp_sum(s);
  if ((tid & 31) == 0) red[tid >> 5] = s;
  __syncthreads();
  if (tid == 0) {
    double v = 0.0;
    for (int w = 0; w < 8; w++) v += red[w];
    out[t] = v;
  }
}

// Row abs-sums of the rank's panels for ||M||_inf (symmetric, lower stored):
// rs[i] = sum over the rank's columns c <= i of |M(i, c)|  +  (column i local:
// sum_{r > i} |M(r, i)|).  One thread per row; fixed order.
__global__ void __launch_bounds__(256) k_dp_rowabs(int64_t N, const double* __restrict__ C, int64_t ldc,
                                                   const int64_t* kq, const int* wq, int nq, double* rs) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  double s = 0.0;
  for (int q = 0; q < nq; q++) {
    const double* Cq = C + (int64_t)q * DB * ldc;
    for (int c = 0; c < wq[q]; c++) {
      const int64_t gc = kq[q] + c;
      if (gc < i) s += fabs(Cq[i + (int64_t)c * ldc]);
      else if (gc == i) {
        s += fabs(Cq[i + (int64_t)c * ldc]);
        for (int64_t r = i + 1; r < N; r++) s += fabs(Cq[r + (int64_t)c * ldc]);
      }
    }
  }
  rs[i] = s;
}
}  // namespace

extern "C" int mds_dist_panel(int64_t n, int nb, const double* A, int64_t lda, double* L, double* W, int64_t ldl,
                              double* d, double* cmax, double* parts, int64_t nparts_cap, double tol,
                              int32_t* accepted, long long* inertia, void* stream) {
  if (n < 1 || nb < 1 || nb > DB || nb > n || !A || !L || !W || !d || !cmax || !parts || !accepted || !inertia ||
      lda < n || ldl < n)
    return MDS_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t rows = n - nb;
  const int nparts = (int)((rows + 127) / 128);
  if (nparts > nparts_cap) return MDS_ERR_WORKSPACE;
  MDS_LAUNCH(PC_PANEL_DIAG, s, (k_dp_f1<<<1, 256, 0, s>>>(nb, A, lda, L, W, ldl, d, cmax)));
  if (nparts > 0) MDS_LAUNCH(PC_PANEL_TRSM, s, (k_dp_f2<DB><<<nparts, 128, 0, s>>>(n, nb, A, lda, L, W, ldl, d, parts)));
  MDS_LAUNCH(PC_PANEL_SLOW, s, (k_dp_accept<<<1, DB, 0, s>>>(nb, d, cmax, parts, nparts, tol, accepted, inertia)));
  return MDS_OK;
}

extern "C" int mds_dist_update(int64_t N, int64_t k0, int nb, const double* L, const double* W, int64_t ldl, double* C,
                               int64_t ldc, const int64_t* kq, const int* wq, int nq, int64_t max_rows, void* stream) {
  if (N < 0 || k0 < 0 || nb < 1 || nb > DB || nq < 0 || (nq > 0 && (!L || !W || !C || !kq || !wq))) return MDS_ERR_ARG;
  if (nq == 0 || max_rows <= 0) return MDS_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const unsigned gx = (unsigned)((max_rows + DB - 1) / DB);
  MDS_LAUNCH(PC_UPDATE, s, (k_dp_update<<<dim3(gx, (unsigned)nq), 256, 0, s>>>(N, k0, nb, L, W, ldl, C, ldc, kq, wq)));
  return MDS_OK;
}

extern "C" int mds_dist_trsv64(int nb, const double* L, int64_t ldl, double* y, int mode, void* stream) {
  if (nb < 1 || nb > DB || !L || !y || (mode != 0 && mode != 1)) return MDS_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  MDS_LAUNCH(PC_SOLVE_FWD, s, (k_dp_trsv64<<<1, DB, 0, s>>>(nb, L, ldl, y, mode)));
  return MDS_OK;
}

extern "C" int mds_dist_gemv_n(int64_t r0, int64_t r1, int nb, const double* L, int64_t ldl, const double* y,
                               double* acc, void* stream) {
  if (nb < 1 || nb > DB || r0 < 0 || !L || !y || !acc) return MDS_ERR_ARG;
  if (r1 <= r0) return MDS_OK;
  cudaStream_t s = (cudaStream_t)stream;
  MDS_LAUNCH(PC_SOLVE_FWD, s, (k_dp_gemv_n<<<(unsigned)((r1 - r0 + 255) / 256), 256, 0, s>>>(r0, r1, nb, L, ldl, y, acc)));
  return MDS_OK;
}

extern "C" int mds_dist_gemv_t(int64_t r0, int64_t r1, int nb, const double* L, int64_t ldl, const double* x,
                               double* out, void* stream) {
  if (nb < 1 || nb > DB || r0 < 0 || !L || !x || !out) return MDS_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  MDS_LAUNCH(PC_SOLVE_BWD, s, (k_dp_gemv_t<<<(unsigned)nb, 256, 0, s>>>(r0, r1, L, ldl, x, out)));
  return MDS_OK;
}

extern "C" int mds_dist_rowabs(int64_t N, const double* C, int64_t ldc, const int64_t* kq, const int* wq, int nq,
                               double* rs, void* stream) {
  if (N < 0 || nq < 0 || !rs || (nq > 0 && (!C || !kq || !wq))) return MDS_ERR_ARG;
  if (N == 0) return MDS_OK;
  cudaStream_t s = (cudaStream_t)stream;
  MDS_LAUNCH(PC_ANORM, s, (k_dp_rowabs<<<(unsigned)((N + 255) / 256), 256, 0, s>>>(N, C, ldc, kq, wq, nq, rs)));
  return MDS_OK;
}
