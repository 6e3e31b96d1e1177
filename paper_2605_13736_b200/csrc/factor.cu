// factor.cu — mds_factor: blocked FP64 Bunch-Kaufman LDL^T with inertia
// (K4; alpha = (1+sqrt 17)/8), designed for sm_100a.
//
// Right-looking, LAPACK-dlasyf-style panels of width NB with a W = L*D work
// panel, followed by a rank-kb trailing update C -= L21 * W21^T that runs on
// the FP64 tensor cores (mma.sync m8n8k4 f64 -> SASS DMMA; there is no FP64
// tcgen05 kind on Blackwell).  Each panel first tries a SPECULATIVE fast path:
//   F1 k_panel_diag   one CTA factors the NB x NB diagonal block without
//                     pivoting (in shared memory),
//   F2 k_panel_trsm   all SMs form W21 = A21 L11^{-T} (the fully updated
//                     panel columns) and the per-column BK colmax,
//   F3 k_panel_accept accepts the longest prefix of columns that pass BK's
//                     1x1-no-interchange test |d_k| >= alpha*colmax_k (the test
//                     BK itself applies to exactly these numbers), stores L.
// Columns after the first failing one are recomputed by the exact sequential
// BK panel (F4 k_panel_slow, dlasyf semantics: rowmax, 1x1 / 2x2 / interchange).
// So the pivot sequence is Bunch-Kaufman's; only the operation order differs
// (reading R7: parity is on inertia and x).  Quasi-definite KKT matrices take
// the fast path almost always, so the per-column global pivot search costs
// one grid-wide reduction per PANEL instead of one barrier per column.
//
// Panel control lives on the device (FCtl cursor), so the host launch
// sequence is fixed and the whole factorization is CUDA-graph capturable.
// Storage: L of each panel is kept in panel-end row order (dlasyf without its
// final "undo"); k_factor_finalize converts to the explicit-permutation form
// P M P^T = L D L^T consumed by mds_solve.
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace {
constexpr int NB = 64;              // panel width
constexpr int WCOLS = NB + 1;       // W work panel columns (+1 for the 2x2 candidate)
constexpr double ALPHA_BK = 0.64038820320220756872767623199676;  // (1+sqrt(17))/8

struct FCtl {
  int k0;          // first column of the current panel
  int kb;          // columns finished in the current panel
  int nbp;         // width of the current panel's diagonal block
  int npanel;      // panels started
  int nswap;       // interchanges performed (kp != kk)
  int abort;       // non-finite input: nothing is factored
  int pad[2];
  double anorm, tol;
  long long inertia[3];
  unsigned long long colmax[NB];   // bit patterns of non-negative doubles (atomicMax-able)
  double d[NB];
};

struct FWork {
  FCtl* ctl;
  int* panel_start;   // [N+1]
  int* sw;            // [N]  kp of the interchange whose kk is this column, else -1
  int* bt;            // [N]  0: 1x1, 1: first of 2x2, 2: second of 2x2
  int* rho;           // [N]
  int* rhoinv;        // [N]
  double* rowsum;     // [N]
  double* Lblk;       // [NB*NB]
  double* W;          // [ldw * WCOLS]
  int64_t ldw;
};

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

FWork carve(void* work, int64_t N, size_t* total) {
  FWork f;
  size_t off = 0;
  char* base = reinterpret_cast<char*>(work);
  auto take = [&](size_t bytes) { char* p = base + off; off = align_up(off + bytes, 256); return p; };
  f.ctl = reinterpret_cast<FCtl*>(take(sizeof(FCtl)));
  f.panel_start = reinterpret_cast<int*>(take(sizeof(int) * (N + 1)));
  f.sw = reinterpret_cast<int*>(take(sizeof(int) * N));
  f.bt = reinterpret_cast<int*>(take(sizeof(int) * N));
  f.rho = reinterpret_cast<int*>(take(sizeof(int) * N));
  f.rhoinv = reinterpret_cast<int*>(take(sizeof(int) * N));
  f.rowsum = reinterpret_cast<double*>(take(sizeof(double) * N));
  f.Lblk = reinterpret_cast<double*>(take(sizeof(double) * NB * NB));
  f.ldw = align_up(std::max<int64_t>(N, 1), 4);
  f.W = reinterpret_cast<double*>(take(sizeof(double) * f.ldw * WCOLS));
  if (total) *total = off;
  return f;
}

__device__ __forceinline__ unsigned long long dbits(double v) { return (unsigned long long)__double_as_longlong(v); }
__device__ __forceinline__ double bitsd(unsigned long long b) { return __longlong_as_double((long long)b); }

// ---------------------------------------------------------------------------
__global__ void k_factor_init(FCtl* ctl, double zero_tol) {
  ctl->tol = zero_tol;
}

// ||M||_inf (row abs-sums via symmetry, lower storage) + non-finite scan.
// One CTA per 32x32 lower tile; row partials atomically added to rowsum.
__global__ void __launch_bounds__(256) k_anorm_tiles(int64_t N, const double* __restrict__ A, int64_t lda,
                                                     double* rowsum, FCtl* ctl, int32_t* status) {
  const int64_t nt = (N + 31) / 32;
  const int64_t x = blockIdx.x;
  int64_t bi = (int64_t)((sqrt(8.0 * (double)x + 1.0) - 1.0) * 0.5);
  while (bi * (bi + 1) / 2 > x) bi--;
  while ((bi + 1) * (bi + 2) / 2 <= x) bi++;
  const int64_t bj = x - bi * (bi + 1) / 2;
  if (bi >= nt) return;
  __shared__ double tile[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // 32 x 8
  bool bad = false;
  for (int yy = ty; yy < 32; yy += 8) {
    const int64_t i = bi * 32 + tx, j = bj * 32 + yy;
    double v = 0.0;
    if (i < N && j < N && i >= j) {
      v = A[i + j * lda];
      if (!isfinite(v)) bad = true;
      v = fabs(v);
    }
    tile[yy][tx] = v;   // tile[col][row]
  }
  if (__syncthreads_or(bad)) {
    if (threadIdx.x == 0) { mds_set_status(status, MDS_ERR_NONFINITE); ctl->abort = 1; }
    return;
  }
  if (threadIdx.x < 32) {
    // row sums (row i = bi*32+tx) over tile columns
    double s = 0.0;
    for (int c = 0; c < 32; c++) s += tile[c][threadIdx.x];
    const int64_t i = bi * 32 + threadIdx.x;
    if (i < N && s != 0.0) atomicAdd(&rowsum[i], s);
  } else if (threadIdx.x < 64) {
    // column sums excluding the diagonal (they are row j's upper part)
    const int c = threadIdx.x - 32;
    double s = 0.0;
    for (int r = 0; r < 32; r++) {
      const int64_t i = bi * 32 + r, j = bj * 32 + c;
      if (i > j) s += tile[c][r];
    }
    const int64_t j = bj * 32 + c;
    if (j < N && s != 0.0) atomicAdd(&rowsum[j], s);
  }
}

__global__ void __launch_bounds__(1024) k_anorm_final(int64_t N, const double* rowsum, FCtl* ctl) {
  double m = 0.0;
  for (int64_t i = threadIdx.x; i < N; i += blockDim.x) m = fmax(m, rowsum[i]);
  m = warp_max(m);
  __shared__ double sh[32];
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); w++) a = fmax(a, sh[w]);
    ctl->anorm = a;
    if (ctl->tol < 0.0) ctl->tol = (double)N * 2.220446049250313e-16 * a;
  }
}

// ---------------------------------------------------------------------------
// F1: unpivoted LDL^T of the NB x NB diagonal block in shared memory.
// Leaves W11 (updated, unscaled columns) in W, L11 in Lblk, d and the in-block
// part of colmax in ctl.  A is NOT modified (rejected columns need originals).
__global__ void __launch_bounds__(256) k_panel_diag(int64_t N, const double* __restrict__ A, int64_t lda,
                                                    FWork f) {
  FCtl* ctl = f.ctl;
  if (ctl->abort) return;
  __shared__ double Ad[NB * (NB + 1)];    // column-major, stride NB+1
  __shared__ int s_k0;
  if (threadIdx.x == 0) s_k0 = ctl->k0 + ctl->kb;
  __syncthreads();
  const int64_t k0 = s_k0;
  if (k0 >= N) {
    if (threadIdx.x == 0) { ctl->k0 = (int)N; ctl->kb = 0; ctl->nbp = 0; }
    return;
  }
  const int nbp = (int)((N - k0) < NB ? (N - k0) : NB);
  constexpr int S = NB + 1;
  for (int idx = threadIdx.x; idx < nbp * nbp; idx += blockDim.x) {
    const int i = idx % nbp, j = idx / nbp;
    if (i >= j) Ad[j * S + i] = A[(k0 + i) + (k0 + j) * lda];
  }
  __syncthreads();
  for (int j = 0; j < nbp; j++) {
    const double d = Ad[j * S + j];
    const double r1 = (d != 0.0) ? 1.0 / d : 0.0;
    // A22 -= (a r1) a^T over the trailing block (lower), a = column j (unscaled)
    const int m = nbp - j - 1;
    for (int idx = threadIdx.x; idx < m * m; idx += blockDim.x) {
      const int r = j + 1 + idx % m, c = j + 1 + idx / m;
      if (r >= c) Ad[c * S + r] -= (Ad[j * S + r] * r1) * Ad[j * S + c];
    }
    __syncthreads();
  }
  // W11 = updated columns (Ad lower), L11 = W11 * r1, in-block colmax, d
  for (int idx = threadIdx.x; idx < nbp * nbp; idx += blockDim.x) {
    const int r = idx % nbp, j = idx / nbp;
    if (r >= j) {
      const double wv = Ad[j * S + r];
      f.W[(k0 + r) + j * f.ldw] = wv;
      const double d = Ad[j * S + j];
      const double r1 = (d != 0.0) ? 1.0 / d : 0.0;
      f.Lblk[r + j * NB] = (r == j) ? 1.0 : wv * r1;
    } else {
      f.Lblk[r + j * NB] = 0.0;
    }
  }
  if (threadIdx.x < NB) {
    const int j = threadIdx.x;
    if (j < nbp) {
      double cm = 0.0;
      for (int r = j + 1; r < nbp; r++) cm = fmax(cm, fabs(Ad[j * S + r]));
      ctl->colmax[j] = dbits(cm);
      ctl->d[j] = Ad[j * S + j];
    }
  }
  if (threadIdx.x == 0) {
    ctl->k0 = (int)k0;
    ctl->kb = 0;
    ctl->nbp = nbp;
    f.panel_start[ctl->npanel] = (int)k0;
    ctl->npanel += 1;
  }
}

// F2: W21 = A21 L11^{-T} (forward substitution per row, registers) and the
// colmax of every panel column over rows below the diagonal block.
__global__ void __launch_bounds__(256) k_panel_trsm(int64_t N, const double* __restrict__ A, int64_t lda, FWork f) {
  FCtl* ctl = f.ctl;
  if (ctl->abort) return;
  const int nbp = ctl->nbp;
  const int64_t k0 = ctl->k0;
  if (nbp == 0) return;
  const int64_t rbase = k0 + nbp + (int64_t)blockIdx.x * 256;
  if (rbase >= N) return;
  __shared__ double Ls[NB * NB];    // Ls[t*NB + j] = L11[j, t]
  __shared__ double wmax[8][NB];
  for (int idx = threadIdx.x; idx < NB * NB; idx += 256) {
    const int j = idx % NB, t = idx / NB;
    Ls[idx] = (j < nbp && t < nbp) ? f.Lblk[j + t * NB] : 0.0;
  }
  __syncthreads();
  const int64_t r = rbase + threadIdx.x;
  const bool live = r < N;
  double x[NB];
#pragma unroll
  for (int t = 0; t < NB; t++) x[t] = (live && t < nbp) ? A[r + (k0 + t) * lda] : 0.0;
#pragma unroll
  for (int j = 1; j < NB; j++) {
    double s = x[j];
#pragma unroll
    for (int t = 0; t < j; t++) s -= x[t] * Ls[t * NB + j];
    x[j] = s;
  }
  if (live) {
#pragma unroll
    for (int t = 0; t < NB; t++)
      if (t < nbp) f.W[r + t * f.ldw] = x[t];
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int t = 0; t < NB; t++) {
    double v = warp_max(fabs(x[t]));
    if (lane == 0) wmax[warp][t] = v;
  }
  __syncthreads();
  if (threadIdx.x < nbp) {
    double v = 0.0;
    for (int w = 0; w < 8; w++) v = fmax(v, wmax[w][threadIdx.x]);
    atomicMax(&ctl->colmax[threadIdx.x], dbits(v));
  }
}

// F3: accept the longest prefix of columns that pass BK's 1x1-no-interchange
// test, write L (= W * 1/d) and D for them; counts inertia; sets ctl->kb.
__global__ void __launch_bounds__(256) k_panel_accept(int64_t N, double* __restrict__ A, int64_t lda, FWork f,
                                                      int32_t* piv) {
  FCtl* ctl = f.ctl;
  if (ctl->abort) return;
  const int nbp = ctl->nbp;
  const int64_t k0 = ctl->k0;
  if (nbp == 0) return;
  __shared__ int s_p;
  __shared__ double s_r1[NB], s_d[NB];
  if (threadIdx.x == 0) {
    int p = 0;
    while (p < nbp) {
      const double d = ctl->d[p], cm = bitsd(ctl->colmax[p]);
      if (!(fabs(d) >= ALPHA_BK * cm)) break;   // (0 >= 0 accepts the exact-zero column)
      p++;
    }
    s_p = p;
  }
  if (threadIdx.x < NB) {
    const double d = (threadIdx.x < nbp) ? ctl->d[threadIdx.x] : 0.0;
    s_d[threadIdx.x] = d;
    s_r1[threadIdx.x] = (d != 0.0) ? 1.0 / d : 0.0;
  }
  __syncthreads();
  const int p = s_p;
  const int64_t r = k0 + (int64_t)blockIdx.x * 256 + threadIdx.x;
  if (r < N) {
    for (int j = 0; j < p; j++) {
      const int64_t k = k0 + j;
      if (r == k) A[r + k * lda] = s_d[j];
      else if (r > k) A[r + k * lda] = f.W[r + j * f.ldw] * s_r1[j];
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const double tol = ctl->tol;
    for (int j = 0; j < p; j++) {
      const double d = s_d[j];
      if (d > tol) ctl->inertia[0]++;
      else if (d < -tol) ctl->inertia[2]++;
      else ctl->inertia[1]++;
      piv[k0 + j] = (int32_t)(k0 + j + 1);
    }
    ctl->kb = p;
  }
}

// F4: exact sequential Bunch-Kaufman panel (LAPACK dlasyf 'L' semantics) for
// the columns the fast path did not accept.  One CTA of 1024 threads; rows
// are strided over threads; W holds updated columns, A holds L for finished
// columns and ORIGINAL (interchanged) values elsewhere.
__device__ __forceinline__ ArgMax block_argmax(ArgMax a, ArgMax* sh) {
  a = warp_argmax(a);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) sh[warp] = a;
  __syncthreads();
  if (warp == 0) {
    ArgMax b = (lane < (int)(blockDim.x >> 5)) ? sh[lane] : ArgMax{-1.0, 0x7fffffff};
    b = warp_argmax(b);
    if (lane == 0) sh[32] = b;
  }
  __syncthreads();
  return sh[32];
}

__global__ void __launch_bounds__(1024) k_panel_slow(int64_t N, double* __restrict__ A, int64_t lda, FWork f,
                                                     int32_t* piv) {
  FCtl* ctl = f.ctl;
  if (ctl->abort) return;
  const int nbp = ctl->nbp;
  const int64_t k0 = ctl->k0;
  int j = ctl->kb;
  if (nbp == 0) return;
  const bool last = (k0 + nbp >= N);
  const int jlim = last ? nbp : nbp - 1;
  if (j >= jlim) return;
  __shared__ double wrow[WCOLS];
  __shared__ ArgMax sh[33];
  double* W = f.W;
  const int64_t ldw = f.ldw;
  const int tid = threadIdx.x, nth = blockDim.x;
  const double tol = ctl->tol;
  while (j < jlim) {
    const int64_t k = k0 + j;
    for (int t = tid; t < j; t += nth) wrow[t] = W[k + t * ldw];
    __syncthreads();
    // W(k:N, j) = A(k:N, k) - L(k:N, panel) * W(k, panel)^T ; argmax below k
    ArgMax am{-1.0, 0x7fffffff};
    for (int64_t r = k + tid; r < N; r += nth) {
      double v = A[r + k * lda];
      for (int t = 0; t < j; t++) v -= A[r + (k0 + t) * lda] * wrow[t];
      W[r + j * ldw] = v;
      if (r > k) am = am_better(am, ArgMax{fabs(v), (int)r});
    }
    am = block_argmax(am, sh);   // contains __syncthreads
    const double absakk = fabs(W[k + j * ldw]);
    const double colmax = (am.v < 0.0) ? 0.0 : am.v;
    const int64_t imax = (am.v < 0.0) ? k : am.i;
    int kstep = 1;
    int64_t kp = k;
    bool zero = false;
    if (fmax(absakk, colmax) == 0.0) {
      zero = true;
    } else if (absakk >= ALPHA_BK * colmax) {
      kp = k;
    } else {
      for (int t = tid; t < j; t += nth) wrow[t] = W[imax + t * ldw];
      __syncthreads();
      // candidate column imax, updated: W(k:N, j+1)
      ArgMax rm{-1.0, 0x7fffffff};
      for (int64_t r = k + tid; r < N; r += nth) {
        double v = (r < imax) ? A[imax + r * lda] : A[r + imax * lda];
        for (int t = 0; t < j; t++) v -= A[r + (k0 + t) * lda] * wrow[t];
        W[r + (j + 1) * ldw] = v;
        if (r != imax) rm = am_better(rm, ArgMax{fabs(v), (int)r});
      }
      rm = block_argmax(rm, sh);
      const double rowmax = (rm.v < 0.0) ? 0.0 : rm.v;
      const double wii = fabs(W[imax + (j + 1) * ldw]);
      if (absakk >= ALPHA_BK * colmax * (colmax / rowmax)) {
        kp = k;
      } else if (wii >= ALPHA_BK * rowmax) {
        kp = imax;
        for (int64_t r = k + tid; r < N; r += nth) W[r + j * ldw] = W[r + (j + 1) * ldw];
        __syncthreads();
      } else {
        kp = imax;
        kstep = 2;
      }
    }
    const int64_t kk = k + kstep - 1;
    if (kp != kk) {
      // symmetric interchange kk <-> kp of the not-yet-factored (original) part
      for (int64_t r = kk + 1 + tid; r < N; r += nth) {
        if (r < kp) A[kp + r * lda] = A[r + kk * lda];
        else if (r > kp) A[r + kp * lda] = A[r + kk * lda];
      }
      if (tid == 0) A[kp + kp * lda] = A[kk + kk * lda];
      // rows kk <-> kp of the panel's finished L columns and of W
      for (int64_t c = k0 + tid; c < kk; c += nth) {
        double t = A[kk + c * lda]; A[kk + c * lda] = A[kp + c * lda]; A[kp + c * lda] = t;
      }
      for (int64_t t = tid; t <= kk - k0; t += nth) {
        double u = W[kk + t * ldw]; W[kk + t * ldw] = W[kp + t * ldw]; W[kp + t * ldw] = u;
      }
      if (tid == 0) { f.sw[kk] = (int)kp; ctl->nswap += 1; }
      __syncthreads();
    }
    if (kstep == 1) {
      const double d = W[k + j * ldw];
      const double r1 = zero ? 0.0 : 1.0 / d;
      for (int64_t r = k + 1 + tid; r < N; r += nth) A[r + k * lda] = zero ? W[r + j * ldw] : W[r + j * ldw] * r1;
      if (tid == 0) {
        A[k + k * lda] = d;
        if (d > tol) ctl->inertia[0]++;
        else if (d < -tol) ctl->inertia[2]++;
        else ctl->inertia[1]++;
        piv[k] = (int32_t)(kp + 1);
        f.bt[k] = 0;
      }
    } else {
      double d21 = W[(k + 1) + j * ldw];
      const double d11 = W[(k + 1) + (j + 1) * ldw] / d21;
      const double d22 = W[k + j * ldw] / d21;
      const double tt = 1.0 / (d11 * d22 - 1.0);
      d21 = tt / d21;
      for (int64_t r = k + 2 + tid; r < N; r += nth) {
        const double wk = W[r + j * ldw], wk1 = W[r + (j + 1) * ldw];
        A[r + k * lda] = d21 * (d11 * wk - wk1);
        A[r + (k + 1) * lda] = d21 * (d22 * wk1 - wk);
      }
      if (tid == 0) {
        A[k + k * lda] = W[k + j * ldw];
        A[(k + 1) + k * lda] = W[(k + 1) + j * ldw];
        A[(k + 1) + (k + 1) * lda] = W[(k + 1) + (j + 1) * ldw];
        ctl->inertia[0]++;
        ctl->inertia[2]++;
        piv[k] = piv[k + 1] = (int32_t)(-(kp + 1));
        f.bt[k] = 1;
        f.bt[k + 1] = 2;
      }
    }
    __syncthreads();
    j += kstep;
  }
  if (tid == 0) ctl->kb = j;
}

// ---------------------------------------------------------------------------
// Trailing update C -= L21 * W21^T on the lower triangle, FP64 tensor cores.
// 64x64 tile per CTA, 4 warps of 32x32, mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4),
// full K (= kb <= NB) staged in shared memory, C held in registers.
constexpr int UT = 64;          // tile edge
constexpr int US = UT + 4;      // smem row stride (conflict-free fragment loads)

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(128) k_update(int64_t N, double* __restrict__ A, int64_t lda, FWork f) {
  FCtl* ctl = f.ctl;
  if (ctl->abort) return;
  const int64_t k0 = ctl->k0;
  const int kb = ctl->kb;
  const int64_t s = k0 + kb;
  const int64_t n2 = N - s;
  if (n2 <= 0 || kb <= 0) return;
  const int64_t nt = (n2 + UT - 1) / UT;
  const int64_t x = blockIdx.x;
  if (x >= nt * (nt + 1) / 2) return;
  int64_t bi = (int64_t)((sqrt(8.0 * (double)x + 1.0) - 1.0) * 0.5);
  while (bi * (bi + 1) / 2 > x) bi--;
  while ((bi + 1) * (bi + 2) / 2 <= x) bi++;
  const int64_t bj = x - bi * (bi + 1) / 2;
  const int64_t R0 = s + bi * UT, C0 = s + bj * UT;
  extern __shared__ double sm[];
  double* Ls = sm;                 // [t][row]
  double* Ws = sm + NB * US;       // [t][col]
  const int kp4 = (kb + 3) & ~3;
  for (int idx = threadIdx.x; idx < UT * kp4; idx += 128) {
    const int i = idx % UT, t = idx / UT;
    const bool tin = t < kb;
    Ls[t * US + i] = (tin && R0 + i < N) ? A[(R0 + i) + (k0 + t) * lda] : 0.0;
    Ws[t * US + i] = (tin && C0 + i < N) ? f.W[(C0 + i) + t * f.ldw] : 0.0;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
  const int g = lane >> 2, q = lane & 3;
  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; a++)
#pragma unroll
    for (int b = 0; b < 4; b++)
#pragma unroll
      for (int e = 0; e < 2; e++) {
        const int64_t row = R0 + wm + 8 * a + g, col = C0 + wn + 8 * b + 2 * q + e;
        acc[a][b][e] = (row < N && col < N) ? A[row + col * lda] : 0.0;
      }
  __syncthreads();
  for (int t0 = 0; t0 < kp4; t0 += 4) {
    double av[4], bv[4];
#pragma unroll
    for (int a = 0; a < 4; a++) av[a] = -Ls[(t0 + q) * US + wm + 8 * a + g];
#pragma unroll
    for (int b = 0; b < 4; b++) bv[b] = Ws[(t0 + q) * US + wn + 8 * b + g];
#pragma unroll
    for (int a = 0; a < 4; a++)
#pragma unroll
      for (int b = 0; b < 4; b++) dmma(acc[a][b][0], acc[a][b][1], av[a], bv[b]);
  }
#pragma unroll
  for (int a = 0; a < 4; a++)
#pragma unroll
    for (int b = 0; b < 4; b++)
#pragma unroll
      for (int e = 0; e < 2; e++) {
        const int64_t row = R0 + wm + 8 * a + g, col = C0 + wn + 8 * b + 2 * q + e;
        if (row < N && col < N && row >= col) A[row + col * lda] = acc[a][b][e];
      }
}

// ---------------------------------------------------------------------------
// Finalize: inertia out; convert panel-end-order L to the explicit permutation
// form by applying every later panel's interchanges to earlier panels' rows
// (only if any interchange happened); final permutation + 2x2 flags into piv[N..2N).
__global__ void k_factor_finalize(int64_t N, double* __restrict__ A, int64_t lda, FWork f, int32_t* piv,
                                  mds_inertia* inertia_out) {
  cg::grid_group grid = cg::this_grid();
  FCtl* ctl = f.ctl;
  const int64_t gtid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t gth = (int64_t)gridDim.x * blockDim.x;
  if (gtid == 0 && inertia_out) {
    inertia_out->pos = ctl->inertia[0];
    inertia_out->zero = ctl->inertia[1];
    inertia_out->neg = ctl->inertia[2];
  }
  if (ctl->abort) return;
  for (int64_t i = gtid; i < N; i += gth) { f.rho[i] = (int)i; f.rhoinv[i] = (int)i; }
  const int npan = ctl->npanel;
  const int nswap = ctl->nswap;
  grid.sync();
  if (nswap > 0) {
    for (int q = npan - 1; q >= 0; q--) {
      const int64_t c0 = f.panel_start[q];
      const int64_t c1 = (q + 1 < npan) ? f.panel_start[q + 1] : N;
      const int64_t nr = N - c1, nc = c1 - c0;
      if (nr > 0) {
        for (int64_t idx = gtid; idx < nr * nc; idx += gth) {
          const int64_t i = c1 + idx % nr, c = c0 + idx / nr;
          f.W[i + (c - c0) * f.ldw] = A[(int64_t)f.rho[i] + c * lda];
        }
        grid.sync();
        for (int64_t idx = gtid; idx < nr * nc; idx += gth) {
          const int64_t i = c1 + idx % nr, c = c0 + idx / nr;
          A[i + c * lda] = f.W[i + (c - c0) * f.ldw];
        }
      }
      if (gtid == 0) {
        for (int64_t k = c1 - 1; k >= c0; k--) {
          const int b = f.sw[k];
          if (b >= 0) {
            const int a = (int)k;
            const int ia = f.rhoinv[a], ib = f.rhoinv[b];
            f.rho[ia] = b; f.rho[ib] = a;
            f.rhoinv[a] = ib; f.rhoinv[b] = ia;
          }
        }
      }
      grid.sync();
    }
  }
  for (int64_t i = gtid; i < N; i += gth) {
    piv[N + i] = f.rho[i] | (f.bt[i] << 29);
    if (f.bt[i] == 1) {   // move the 2x2 off-diagonal d21 to the upper slot (i, i+1): L(i+1, i) = 0
      A[i + (i + 1) * lda] = A[(i + 1) + i * lda];
      A[(i + 1) + i * lda] = 0.0;
    }
  }
}
}  // namespace

// read by solve.cu
double* mds_factor_tol_ptr(const void* fwork) {
  return fwork ? &reinterpret_cast<FCtl*>(const_cast<void*>(fwork))->tol : nullptr;
}

extern "C" size_t mds_factor_workspace_size(int64_t N) {
  size_t total = 0;
  carve(nullptr, std::max<int64_t>(N, 1), &total);
  return total;
}

extern "C" int mds_factor(int64_t N, double* M, int64_t ldm, int32_t* piv, double zero_tol,
                          mds_inertia* inertia_dev, mds_inertia* inertia_host, int32_t* status,
                          void* work, size_t work_bytes, void* stream) {
  if (N < 0 || (N > 0 && (!M || !piv)) || ldm < std::max<int64_t>(N, 1)) return MDS_ERR_ARG;
  if (N >= (1 << 29)) return MDS_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  if (N == 0) {
    if (inertia_dev) MDS_CUDA_TRY(cudaMemsetAsync(inertia_dev, 0, sizeof(mds_inertia), st));
    if (inertia_host) { inertia_host->pos = inertia_host->zero = inertia_host->neg = 0; }
    return MDS_OK;
  }
  size_t need = mds_factor_workspace_size(N);
  if (!work || work_bytes < need) return MDS_ERR_WORKSPACE;
  FWork f = carve(work, N, nullptr);
  // zero control + arrays (sw = -1)
  MDS_CUDA_TRY(cudaMemsetAsync(f.ctl, 0, sizeof(FCtl), st));
  MDS_CUDA_TRY(cudaMemsetAsync(f.sw, 0xff, sizeof(int) * N, st));
  MDS_CUDA_TRY(cudaMemsetAsync(f.bt, 0, sizeof(int) * N, st));
  MDS_CUDA_TRY(cudaMemsetAsync(f.rowsum, 0, sizeof(double) * N, st));
  k_factor_init<<<1, 1, 0, st>>>(f.ctl, zero_tol);
  MDS_LAUNCH_CHECK();
  {
    int64_t nt = (N + 31) / 32;
    k_anorm_tiles<<<(unsigned)(nt * (nt + 1) / 2), 256, 0, st>>>(N, M, ldm, f.rowsum, f.ctl, status);
    MDS_LAUNCH_CHECK();
    k_anorm_final<<<1, 1024, 0, st>>>(N, f.rowsum, f.ctl);
    MDS_LAUNCH_CHECK();
  }
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_update, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * NB * US * (int)sizeof(double));
    attr = true;
  }
  const size_t usmem = 2 * NB * US * sizeof(double);
  const int64_t npmax = (N + (NB - 2)) / (NB - 1) + 1;
  for (int64_t p = 0; p < npmax; p++) {
    const int64_t kmin = std::min<int64_t>(p * (NB - 1), N);   // lower bound on this panel's k0
    const int64_t rows = N - kmin;
    if (rows <= 0) break;
    k_panel_diag<<<1, 256, 0, st>>>(N, M, ldm, f);
    MDS_LAUNCH_CHECK();
    const unsigned g256 = (unsigned)std::max<int64_t>(mds_cdiv(rows, 256), 1);
    k_panel_trsm<<<g256, 256, 0, st>>>(N, M, ldm, f);
    MDS_LAUNCH_CHECK();
    k_panel_accept<<<g256, 256, 0, st>>>(N, M, ldm, f, piv);
    MDS_LAUNCH_CHECK();
    k_panel_slow<<<1, 1024, 0, st>>>(N, M, ldm, f, piv);
    MDS_LAUNCH_CHECK();
    const int64_t n2max = std::max<int64_t>(rows - 1, 0);
    const int64_t nt = mds_cdiv(n2max, UT);
    if (nt > 0) {
      k_update<<<(unsigned)(nt * (nt + 1) / 2), 128, usmem, st>>>(N, M, ldm, f);
      MDS_LAUNCH_CHECK();
    }
  }
  {
    int dev = 0, sms = 148, occ = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_factor_finalize, 256, 0);
    int blocks = sms * std::max(1, std::min(occ, 2));
    void* args[] = {&N, &M, &ldm, &f, &piv, &inertia_dev};
    MDS_CUDA_TRY(cudaLaunchCooperativeKernel((void*)k_factor_finalize, blocks, 256, args, 0, st));
  }
  if (inertia_host) {
    if (!inertia_dev) return MDS_ERR_ARG;
    MDS_CUDA_TRY(cudaMemcpyAsync(inertia_host, inertia_dev, sizeof(mds_inertia), cudaMemcpyDeviceToHost, st));
    MDS_CUDA_TRY(cudaStreamSynchronize(st));
  }
  return MDS_OK;
}
