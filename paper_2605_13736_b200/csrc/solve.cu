// solve.cu — mds_solve: x = P^T L^{-T} D^{-1} L^{-1} P rhs_c with mds_factor's
// explicit-permutation factors (K4 solve), then the sparse
// step recovery dx_s = w .* (r_xs - J_s dy) (K2; first block row
// of Eq.(5)).  HBM-bound: L is streamed once per triangular sweep.
//
// Triangular sweeps are single "sync-free" launches: CTA i (row block of 64,
// index taken from an atomic ticket so lower blocks always run first) streams
// its part of L against already-published blocks, then finishes its block.
// The dependent chain between consecutive blocks is one 64x64 GEMV: with
// Binv_i = L_ii^{-1} and G_i = Binv_i L_{i,i-1} precomputed (k_inv_blocks),
//   y_i = Binv_i (b_i - sum_{q<i-1} L_iq y_q) - G_i y_{i-1},
// where the first term is ready before y_{i-1} is.  Published values are
// their own ready flags: the output vectors are pre-filled with an all-ones
// bit pattern (never produced: NaN results are canonicalised on store) and a
// consumer polls the values it needs.
#include <algorithm>

#include "common.cuh"

const int32_t* mds_plan_rowptr(const mds_plan* P);
const int32_t* mds_plan_colidx(const mds_plan* P);
double* mds_factor_tol_ptr(const void* fwork);
size_t mds_factor_ws_stride_bytes(int64_t N);

namespace {
constexpr int TB = 64;        // row block
constexpr int ST = 256;       // threads
constexpr int PERM_MASK = (1 << 29) - 1;

struct SWork {
  double* b;      // [N] P rhs
  double* y;      // [N] forward result, then D^{-1} applied in place (published values, sentinel-filled)
  double* x;      // [N] backward result (published values, sentinel-filled)
  double* binv;   // [nblk][TB*TB] inverses of the unit-lower diagonal blocks (column-major)
  double* gf;     // [nblk][TB*TB] Binv_i L_{i,i-1}            (column-major)
  double* gb;     // [nblk][TB*TB] (L_{i+1,i} Binv_i)^T        (column-major)
  int* tickets;   // [2]
};
constexpr unsigned long long SENT = ~0ull;   // "not yet published" (a NaN payload never stored)

// Batched solves (mds_solve_batched): scenario s = blockIdx.y reads / writes every
// array at base + s * stride (elements; workspace pointers by bytes).  All zero
// for a single system.
struct BStr {
  int64_t ld, piv, rhs, dxy, val, w, rxs, dxs;
  size_t ws, fws;   // solve / factor workspace bytes per scenario
};
template <typename T>
__device__ __forceinline__ T* bsh(T* p, size_t bytes) {
  return reinterpret_cast<T*>(reinterpret_cast<uintptr_t>(p) + bytes * blockIdx.y);
}

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }
SWork carve(void* work, int64_t N, size_t* total) {
  SWork s;
  size_t off = 0;
  char* b = reinterpret_cast<char*>(work);
  auto take = [&](size_t bytes) { char* p = b + off; off = align_up(off + bytes, 256); return p; };
  s.tickets = reinterpret_cast<int*>(take(sizeof(int) * 4));
  s.b = reinterpret_cast<double*>(take(sizeof(double) * std::max<int64_t>(N, 1)));
  s.y = reinterpret_cast<double*>(take(sizeof(double) * std::max<int64_t>(N, 1)));
  s.x = reinterpret_cast<double*>(take(sizeof(double) * std::max<int64_t>(N, 1)));
  s.binv = reinterpret_cast<double*>(take(sizeof(double) * TB * TB * (N / TB + 1)));
  s.gf = reinterpret_cast<double*>(take(sizeof(double) * TB * TB * (N / TB + 1)));
  s.gb = reinterpret_cast<double*>(take(sizeof(double) * TB * TB * (N / TB + 1)));
  if (total) *total = off;
  return s;
}

__device__ __forceinline__ unsigned long long ld_relaxed_u64(const double* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];\n" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// wait until the n published values at p are all present, return them
template <int NV>
__device__ __forceinline__ void poll_values(const double* p, double* out) {
  unsigned long long v[NV];
  bool ready;
  do {
    ready = true;
#pragma unroll
    for (int c = 0; c < NV; c++) {
      v[c] = ld_relaxed_u64(p + c);
      ready &= (v[c] != SENT);
    }
  } while (!ready);
#pragma unroll
  for (int c = 0; c < NV; c++) out[c] = __longlong_as_double((long long)v[c]);
}
// prefetch NV values (may still be sentinels); complete them later with finish_values
template <int NV>
__device__ __forceinline__ void load_values(const double* p, unsigned long long* v) {
#pragma unroll
  for (int c = 0; c < NV; c++) v[c] = ld_relaxed_u64(p + c);
}
template <int NV>
__device__ __forceinline__ void finish_values(const double* p, unsigned long long* v, double* out) {
  bool ready = true;
#pragma unroll
  for (int c = 0; c < NV; c++) ready &= (v[c] != SENT);
  while (!ready) {
    ready = true;
#pragma unroll
    for (int c = 0; c < NV; c++) {
      if (v[c] == SENT) v[c] = ld_relaxed_u64(p + c);
      ready &= (v[c] != SENT);
    }
  }
#pragma unroll
  for (int c = 0; c < NV; c++) out[c] = __longlong_as_double((long long)v[c]);
}
// 16 published values p[0..16) needed by every lane of the warp: lane l fetches
// p[l & 15] only (prefetched raw value `raw`, completed by polling if it was not
// yet published), then the warp exchanges them by shuffles -- 16x fewer polling
// loads on the line the producer is about to write.  `valid` = how many exist.
__device__ __forceinline__ void warp_values16(const double* p, unsigned long long raw, int valid, double* out) {
  const int lane = threadIdx.x & 31, c = lane & 15;
  double mine = 0.0;
  if (c < valid) finish_values<1>(p + c, &raw, &mine);
#pragma unroll
  for (int u = 0; u < 16; u++) out[u] = __shfl_sync(0xffffffffu, mine, u);
}
__device__ __forceinline__ unsigned long long prefetch16(const double* p, int valid) {
  const int c = threadIdx.x & 15;
  return (c < valid) ? ld_relaxed_u64(p + c) : 0ull;
}
__device__ __forceinline__ void publish(double* p, double v) {
  if (v != v) v = __longlong_as_double(0x7ff8000000000000ll);   // canonical NaN, never the sentinel
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;\n" ::"l"(p), "l"((unsigned long long)__double_as_longlong(v)) : "memory");
}

__global__ void k_gather(int64_t N, const int32_t* __restrict__ piv, const double* __restrict__ b,
                         double* __restrict__ bp, double* y, double* x, int* tickets, BStr z) {
  pdl_wait();
  pdl_trigger();
  piv += blockIdx.y * z.piv; b += blockIdx.y * z.rhs;
  bp = bsh(bp, z.ws); y = bsh(y, z.ws); x = bsh(x, z.ws); tickets = bsh(tickets, z.ws);
  if (blockIdx.x == 0 && threadIdx.x < 4) tickets[threadIdx.x] = 0;
  const double sent = __longlong_as_double((long long)SENT);   // "not yet published"
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
    bp[i] = b[piv[N + i] & PERM_MASK];
    y[i] = sent;
    x[i] = sent;
  }
}

// Inverses of the unit-lower TB x TB diagonal blocks of L (one CTA per block,
// row-by-row: Binv[r][c] = -sum_{k=c}^{r-1} L[r][k] Binv[k][c]), and the
// one-step chain operators Gf_i = Binv_i L_{i,i-1}, Gb_i = (L_{i+1,i} Binv_i)^T.
constexpr int TBP = TB + 1;
constexpr int IBSMEM = (2 * TB * TBP + 4 * 16 * 17) * 8;   // L block, Binv, 16x16 temporaries
// G = false (batched per-scenario sweeps: Binv only) compiles without the chain-operator
// GEMMs (one CTA per block and scenario, 2 per SM)
template <bool G>
__global__ void __launch_bounds__(256, G ? 1 : 2) k_inv_blocks(int64_t N, const double* __restrict__ L, int64_t lda,
                                                    double* __restrict__ binv, double* __restrict__ gf,
                                                    double* __restrict__ gb, BStr z) {
  pdl_wait();
  pdl_trigger();
  L += blockIdx.y * z.ld;
  constexpr bool need_g = G;   // (the batched per-scenario sweeps use Binv only)
  binv = bsh(binv, z.ws);
  if (need_g) { gf = bsh(gf, z.ws); gb = bsh(gb, z.ws); }
  extern __shared__ double ism[];
  double* Ls = ism;                      // Ls[k*TBP + r] = L[r][k]  (diagonal block, later the off-diagonal ones)
  double* Bs = ism + TB * TBP;           // Bs[c*TBP + r] = Binv[r][c]
  const int64_t nblk = (N + TB - 1) / TB;
  const int64_t i = blockIdx.x;
  const int64_t r0 = i * TB;
  const int nr = (int)((N - r0) < TB ? (N - r0) : TB);
  // (every block load below keeps a thread's 16 loads in flight at once)
  constexpr int PER = TB * TB / 256;
  {
    double t[PER];
#pragma unroll
    for (int u = 0; u < PER; u++) {
      const int idx = threadIdx.x + u * 256, r = idx % TB, c = idx / TB;
      t[u] = (r < nr && c < nr && r > c) ? L[(r0 + r) + (r0 + c) * lda] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < PER; u++) {
      const int idx = threadIdx.x + u * 256, r = idx % TB, c = idx / TB;
      Ls[c * TBP + r] = t[u];
      Bs[c * TBP + r] = (r == c) ? 1.0 : 0.0;
    }
  }
  __syncthreads();
  // blocked inversion of the unit-lower block: (1) the four 16x16 diagonal
  // blocks, one warp each (lane c < 16 owns column c, right-looking so each
  // row's update is one FMA); (2) off-diagonal 16x16 blocks by distance dd:
  // Binv_{bi,bj} = -Binv_{bi,bi} sum_{k=bj}^{bi-1} L_{bi,k} Binv_{k,bj}.
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp < 4 && lane < 16) {
    const int o = warp * 16, c = lane;
    double xv[16];
#pragma unroll
    for (int rr = 0; rr < 16; rr++) xv[rr] = (rr == c) ? 1.0 : 0.0;
#pragma unroll
    for (int kk = 0; kk < 15; kk++) {
      const double xk = xv[kk];
#pragma unroll
      for (int rr = kk + 1; rr < 16; rr++) xv[rr] = fma(-Ls[(o + kk) * TBP + o + rr], xk, xv[rr]);
    }
#pragma unroll
    for (int rr = 0; rr < 16; rr++) Bs[(o + c) * TBP + o + rr] = xv[rr];   // (zero above the diagonal)
  }
  __syncthreads();
  {
    double* Ts = Bs + TB * TBP;          // temp 16x16 blocks (third buffer)
    const int er = threadIdx.x & 15, ec = threadIdx.x >> 4;
    for (int dd = 1; dd < 4; dd++) {
      for (int bj = 0; bj + dd < 4; bj++) {
        const int bi = bj + dd;
        double t = 0.0;
        for (int kk = bj * 16; kk < bi * 16; kk++) t = fma(Ls[kk * TBP + bi * 16 + er], Bs[(bj * 16 + ec) * TBP + kk], t);
        Ts[(bj * 16 + ec) * 17 + er] = t;
      }
      __syncthreads();
      for (int bj = 0; bj + dd < 4; bj++) {
        const int bi = bj + dd;
        double t = 0.0;
#pragma unroll
        for (int kk = 0; kk < 16; kk++) t = fma(Bs[(bi * 16 + kk) * TBP + bi * 16 + er], Ts[(bj * 16 + ec) * 17 + kk], t);
        Bs[(bj * 16 + ec) * TBP + bi * 16 + er] = -t;
      }
      __syncthreads();
    }
  }
  double* out = binv + (size_t)i * TB * TB;
  for (int idx = threadIdx.x; idx < TB * TB; idx += blockDim.x) {
    const int r = idx % TB, cc = idx / TB;
    out[idx] = Bs[cc * TBP + r];
  }
  if (!need_g) return;
  // thread (r = tid & 63, column group cg = tid >> 6) computes 16 outputs of each G
  const int r = threadIdx.x & (TB - 1), cg = threadIdx.x >> 6;
  if (i >= 1) {
    // Gf[r][c] = sum_k Binv[r][k] L_{i,i-1}[k][c]
    __syncthreads();
#pragma unroll
    for (int h = 0; h < PER; h += PER / 2) {   // two halves of 8 loads in flight (no spills)
      double t[PER / 2];
#pragma unroll
      for (int u = 0; u < PER / 2; u++) {
        const int idx = threadIdx.x + (h + u) * 256, rr = idx % TB, c = idx / TB;
        t[u] = (rr < nr) ? L[(r0 + rr) + (r0 - TB + c) * lda] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < PER / 2; u++) {
        const int idx = threadIdx.x + (h + u) * 256, rr = idx % TB, c = idx / TB;
        Ls[c * TBP + rr] = t[u];
      }
    }
    __syncthreads();
    double acc[16];
#pragma unroll
    for (int u = 0; u < 16; u++) acc[u] = 0.0;
    for (int k = 0; k < TB; k++) {
      const double bk = Bs[k * TBP + r];
#pragma unroll
      for (int u = 0; u < 16; u++) acc[u] += bk * Ls[(cg * 16 + u) * TBP + k];
    }
    double* go = gf + (size_t)i * TB * TB;
#pragma unroll
    for (int u = 0; u < 16; u++) go[r + (cg * 16 + u) * TB] = acc[u];
  }
  if (i + 1 < nblk) {
    // Gb[c][k] = sum_m L_{i+1,i}[k][m] Binv[m][c]   (thread: c = r, k = cg*16+u)
    const int nr1 = (int)((N - r0 - TB) < TB ? (N - r0 - TB) : TB);
    __syncthreads();
#pragma unroll
    for (int h = 0; h < PER; h += PER / 2) {
      double t[PER / 2];
#pragma unroll
      for (int u = 0; u < PER / 2; u++) {
        const int idx = threadIdx.x + (h + u) * 256, kk = idx % TB, m = idx / TB;
        t[u] = (kk < nr1 && m < nr) ? L[(r0 + TB + kk) + (r0 + m) * lda] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < PER / 2; u++) {
        const int idx = threadIdx.x + (h + u) * 256, kk = idx % TB, m = idx / TB;
        Ls[m * TBP + kk] = t[u];
      }
    }
    __syncthreads();
    double acc[16];
#pragma unroll
    for (int u = 0; u < 16; u++) acc[u] = 0.0;
    for (int m = 0; m < TB; m++) {
      const double bmc = Bs[r * TBP + m];   // Binv[m][c=r]
#pragma unroll
      for (int u = 0; u < 16; u++) acc[u] += Ls[m * TBP + cg * 16 + u] * bmc;
    }
    double* go = gb + (size_t)i * TB * TB;
#pragma unroll
    for (int u = 0; u < 16; u++) go[r + (cg * 16 + u) * TB] = acc[u];   // Gb[c=r][k] at (r, k) column-major
  }
}

// Binv_i and G_i into shared memory with all of a thread's 32 loads in flight at
// once (a load-store loop waits out one round trip per element pair)
__device__ __forceinline__ void stage_chain_ops(double* Bs, double* Gs, const double* __restrict__ bsrc,
                                                const double* __restrict__ gsrc, bool has_g) {
  constexpr int PER = TB * TB / ST;
  double tb[PER], tg[PER];
#pragma unroll
  for (int u = 0; u < PER; u++) {
    const int idx = threadIdx.x + u * ST;
    tb[u] = bsrc[idx];
    tg[u] = has_g ? gsrc[idx] : 0.0;
  }
#pragma unroll
  for (int u = 0; u < PER; u++) {
    const int idx = threadIdx.x + u * ST;
    Bs[idx] = tb[u];
    Gs[idx] = tg[u];
  }
}

// forward: L y = b (unit lower; 2x2 D off-diagonals were moved out of L by the factor).
constexpr int SWSMEM = 2 * TB * TB * 8;   // Binv_i and G_i in shared memory
__global__ void __launch_bounds__(ST) k_trsv_fwd(int64_t N, const double* __restrict__ L, int64_t lda,
                                                 const double* __restrict__ b, double* y,
                                                 const double* __restrict__ binv, const double* __restrict__ gf,
                                                 int* ticket, BStr z) {
  pdl_wait();
  pdl_trigger();
  L += blockIdx.y * z.ld;
  b = bsh(b, z.ws); y = bsh(y, z.ws); binv = bsh(binv, z.ws); gf = bsh(gf, z.ws); ticket = bsh(ticket, z.ws);
  extern __shared__ double fsm[];
  double* Bs = fsm;             // Binv_i, column-major
  double* Gs = fsm + TB * TB;   // Gf_i, column-major
  __shared__ int s_i;
  __shared__ double part[ST / TB][TB];
  __shared__ double v[TB];
  __shared__ double cvec[TB];
  if (threadIdx.x == 0) s_i = atomicAdd(ticket, 1);
  __syncthreads();
  const int64_t i = s_i;
  const int64_t r0 = i * TB;
  const int nr = (int)((N - r0) < TB ? (N - r0) : TB);
  const int r = threadIdx.x & (TB - 1), cgp = threadIdx.x / TB;   // 4 column groups of 16
  stage_chain_ops(Bs, Gs, binv + (size_t)i * TB * TB, gf + (size_t)i * TB * TB, i >= 1);
  const double bi = (threadIdx.x < TB && r < nr) ? b[r0 + r] : 0.0;   // off the chain
  double acc = 0.0;
  double lv[16], ln[16];
  const double* Lr = L + (r0 + r);
  auto loadL = [&](int64_t q, double* dst) {
    const int64_t c0 = q * TB + cgp * 16;
#pragma unroll
    for (int c = 0; c < 16; c++) dst[c] = (r < nr) ? Lr[(c0 + c) * lda] : 0.0;
  };
  const int64_t qend = i - 1;   // blocks streamed here; block i-1 goes through G_i
  // y_q is prefetched together with L's block q (one block ahead), so a published
  // value costs no extra round trip; only values not yet published are polled
  unsigned long long yv = 0ull, yn = 0ull;
  if (qend > 0) { loadL(0, lv); yv = prefetch16(y + cgp * 16, 16); }
  for (int64_t q = 0; q < qend; q++) {
    if (q + 1 < qend) { loadL(q + 1, ln); yn = prefetch16(y + (q + 1) * TB + cgp * 16, 16); }
    double yq[16];
    warp_values16(y + q * TB + cgp * 16, yv, 16, yq);
#pragma unroll
    for (int c = 0; c < 16; c++) acc += lv[c] * yq[c];
#pragma unroll
    for (int c = 0; c < 16; c++) lv[c] = ln[c];
    yv = yn;
  }
  part[cgp][r] = acc;
  __syncthreads();
  if (threadIdx.x < TB) {
    const int rr = threadIdx.x;
    v[rr] = (rr < nr) ? bi - (part[0][rr] + part[1][rr] + part[2][rr] + part[3][rr]) : 0.0;
  }
  __syncthreads();
  // c_i = Binv_i v
  double sacc = 0.0;
#pragma unroll
  for (int c = 0; c < 16; c++) {
    const int cc = cgp * 16 + c;
    sacc += Bs[r + cc * TB] * v[cc];
  }
  __syncthreads();
  part[cgp][r] = sacc;
  __syncthreads();
  if (threadIdx.x < TB) {
    const int rr = threadIdx.x;
    cvec[rr] = part[0][rr] + part[1][rr] + part[2][rr] + part[3][rr];
  }
  __syncthreads();
  // the chain step: y_i = c_i - G_i y_{i-1}
  double g = 0.0;
  if (i >= 1) {
    double yp[16];
    const double* pp = y + (i - 1) * TB + cgp * 16;
    warp_values16(pp, prefetch16(pp, 16), 16, yp);
#pragma unroll
    for (int c = 0; c < 16; c++) g += Gs[r + (cgp * 16 + c) * TB] * yp[c];
  }
  part[cgp][r] = g;
  __syncthreads();
  if (threadIdx.x < TB) {
    const int rr = threadIdx.x;
    if (rr < nr) publish(&y[r0 + rr], cvec[rr] - ((part[0][rr] + part[1][rr]) + (part[2][rr] + part[3][rr])));
  }
}

// Batched sweeps (mds_solve_batched): ONE CTA per scenario walks the whole chain, so
// no CTA waits on another (the single-system sweeps above chain 64-row blocks over
// CTAs through published values).  Right-looking over 64-column blocks of L with the
// vector in shared memory: forward, v_b := Binv_b v_b then v_r -= L(r, b) v_b for the
// rows below (L streamed once, coalesced down each column); backward, t = v_b -
// L(rows below, b)^T v, v_b := Binv_b^T t, last block first.  Fixed-order sums.
constexpr int BST = 512;
constexpr int BSMAX = 128 * 1024;   // largest per-scenario vector kept in shared memory (N <= 16384)
__device__ __forceinline__ double red8(double a) {
  a += __shfl_xor_sync(0xffffffffu, a, 1);
  a += __shfl_xor_sync(0xffffffffu, a, 2);
  a += __shfl_xor_sync(0xffffffffu, a, 4);
  return a;
}
__global__ void __launch_bounds__(BST) k_bsolve_fwd(int64_t N, const double* __restrict__ L, int64_t lda,
                                                    const double* __restrict__ b, double* __restrict__ y,
                                                    const double* __restrict__ binv, BStr z) {
  pdl_wait();
  pdl_trigger();
  L += blockIdx.y * z.ld;
  b = bsh(b, z.ws); y = bsh(y, z.ws); binv = bsh(binv, z.ws);
  extern __shared__ double bv[];   // [N]
  const int tid = threadIdx.x;
  for (int64_t i = tid; i < N; i += BST) bv[i] = b[i];
  __syncthreads();
  const int64_t nblk = (N + TB - 1) / TB;
  const int r8 = tid >> 3, part = tid & 7;
  for (int64_t bb = 0; bb < nblk; bb++) {
    const int64_t r0 = bb * TB;
    const int nr = (int)((N - r0) < TB ? (N - r0) : TB);
    // v_b := Binv_b v_b  (row r8, columns 8 part .. 8 part + 7)
    const double* B = binv + (size_t)bb * TB * TB;
    double acc = 0.0;
#pragma unroll
    for (int u = 0; u < 8; u++) {
      const int c = part * 8 + u;
      acc = fma(B[r8 + c * TB], c < nr ? bv[r0 + c] : 0.0, acc);
    }
    acc = red8(acc);
    __syncthreads();
    if (part == 0 && r8 < nr) bv[r0 + r8] = acc;
    __syncthreads();
    // rows below: v_r -= sum_c L(r, r0 + c) v_b[c]
    // (two rows per thread, 16 loads in flight; each row's sum in the same fixed order)
    for (int64_t r = r0 + TB + tid; r < N; r += 2 * BST) {
      const int64_t r2 = r + BST;
      const bool two = r2 < N;
      const double* lr = L + r + r0 * lda;
      const double* lr2 = L + (two ? r2 : r) + r0 * lda;
      double a[8], b8[8];
#pragma unroll
      for (int u = 0; u < 8; u++) a[u] = b8[u] = 0.0;
      int c = 0;
      for (; c + 8 <= nr; c += 8) {
        double l[8], l2[8];
#pragma unroll
        for (int u = 0; u < 8; u++) {
          l[u] = __ldcs(lr + (int64_t)(c + u) * lda);   // (streamed once)
          l2[u] = __ldcs(lr2 + (int64_t)(c + u) * lda);
        }
#pragma unroll
        for (int u = 0; u < 8; u++) {
          a[u] = fma(l[u], bv[r0 + c + u], a[u]);
          b8[u] = fma(l2[u], bv[r0 + c + u], b8[u]);
        }
      }
      for (; c < nr; c++) {
        a[0] = fma(lr[(int64_t)c * lda], bv[r0 + c], a[0]);
        b8[0] = fma(lr2[(int64_t)c * lda], bv[r0 + c], b8[0]);
      }
      bv[r] -= ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
      if (two) bv[r2] -= ((b8[0] + b8[1]) + (b8[2] + b8[3])) + ((b8[4] + b8[5]) + (b8[6] + b8[7]));
    }
    __syncthreads();
  }
  for (int64_t i = tid; i < N; i += BST) y[i] = bv[i];
}

__global__ void __launch_bounds__(BST) k_bsolve_bwd(int64_t N, const double* __restrict__ L, int64_t lda,
                                                    const double* __restrict__ y, double* __restrict__ x,
                                                    const double* __restrict__ binv, BStr z) {
  pdl_wait();
  pdl_trigger();
  L += blockIdx.y * z.ld;
  y = bsh(y, z.ws); x = bsh(x, z.ws); binv = bsh(binv, z.ws);
  extern __shared__ double bv[];   // [N]
  __shared__ double tb[TB];
  const int tid = threadIdx.x;
  for (int64_t i = tid; i < N; i += BST) bv[i] = y[i];
  __syncthreads();
  const int64_t nblk = (N + TB - 1) / TB;
  const int c8 = tid >> 3, sl = tid & 7;
  for (int64_t bb = nblk - 1; bb >= 0; bb--) {
    const int64_t r0 = bb * TB;
    const int nr = (int)((N - r0) < TB ? (N - r0) : TB);
    // t_c = v_b[c] - sum_{rows below} L(r, r0 + c) v_r  (column c8, rows strided by 8 from sl)
    double a0 = 0.0, a1 = 0.0;
    if (c8 < nr) {
      const double* lc = L + (r0 + c8) * lda;
      int64_t r = r0 + TB + sl;
      double a2 = 0.0, a3 = 0.0;
      for (; r + 24 < N; r += 32) {
        const double l0 = __ldcs(lc + r), l1 = __ldcs(lc + r + 8), l2 = __ldcs(lc + r + 16), l3 = __ldcs(lc + r + 24);
        a0 = fma(l0, bv[r], a0);
        a1 = fma(l1, bv[r + 8], a1);
        a2 = fma(l2, bv[r + 16], a2);
        a3 = fma(l3, bv[r + 24], a3);
      }
      for (; r < N; r += 8) a0 = fma(lc[r], bv[r], a0);
      a0 += a2;
      a1 += a3;
    }
    const double dsum = red8(a0 + a1);
    if (sl == 0) tb[c8] = (c8 < nr) ? bv[r0 + c8] - dsum : 0.0;
    __syncthreads();
    // v_b := Binv_b^T t  (Binv^T[r][c] = Binv[c][r])
    const double* B = binv + (size_t)bb * TB * TB;
    double acc = 0.0;
#pragma unroll
    for (int u = 0; u < 8; u++) {
      const int c = sl * 8 + u;
      acc = fma(B[c + c8 * TB], tb[c], acc);
    }
    acc = red8(acc);
    if (sl == 0 && c8 < nr) bv[r0 + c8] = acc;
    __syncthreads();
  }
  for (int64_t i = tid; i < N; i += BST) x[i] = bv[i];
}

// D solve: 1x1 and 2x2 blocks (LAPACK dsytrs scaled 2x2 formula); 2x2 off-diagonal at (k, k+1) (upper slot)
__global__ void k_dsolve(int64_t N, const double* __restrict__ LD, int64_t lda, const int32_t* __restrict__ piv,
                         double* y, const double* tolp, double tolv, int32_t* status, BStr z) {
  pdl_wait();
  pdl_trigger();
  LD += blockIdx.y * z.ld; piv += blockIdx.y * z.piv; y = bsh(y, z.ws);
  if (tolp) tolp = bsh(tolp, z.fws);
  if (status) status += blockIdx.y * (z.ws ? 1 : 0);
  const double tol = tolp ? *tolp : tolv;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < N; k += (int64_t)gridDim.x * blockDim.x) {
    const int bt = (piv[N + k] >> 29) & 3;
    if (bt == 0) {
      const double d = LD[k + k * lda];
      if (!(fabs(d) > tol)) mds_set_status(status, MDS_ERR_SINGULAR);
      y[k] = y[k] / d;
    } else if (bt == 1) {
      const double akm1k = LD[k + (k + 1) * lda];
      const double akm1 = LD[k + k * lda] / akm1k;
      const double ak = LD[(k + 1) + (k + 1) * lda] / akm1k;
      const double denom = akm1 * ak - 1.0;
      const double bkm1 = y[k] / akm1k;
      const double bk = y[k + 1] / akm1k;
      y[k] = (ak * bkm1 - bk) / denom;
      y[k + 1] = (akm1 * bk - bkm1) / denom;
    }
  }
}

// backward: L^T x = z, blocks from the bottom.  CTA i accumulates
// sum_{q>i+1} L[q rows, i cols]^T x_q (threads run down contiguous column
// segments: thread (k, cg) owns row k of every later block and 16 columns),
// then x_i = Binv_i^T (z_i - acc) - Gb_i x_{i+1}.
__global__ void __launch_bounds__(ST) k_trsv_bwd(int64_t N, const double* __restrict__ L, int64_t lda,
                                                 const double* __restrict__ z, double* x,
                                                 const double* __restrict__ binv, const double* __restrict__ gb,
                                                 int* ticket, BStr zs) {
  pdl_wait();
  pdl_trigger();
  L += blockIdx.y * zs.ld;
  z = bsh(z, zs.ws); x = bsh(x, zs.ws); binv = bsh(binv, zs.ws); gb = bsh(gb, zs.ws); ticket = bsh(ticket, zs.ws);
  extern __shared__ double fsm[];
  double* Bs = fsm;             // Binv_i, column-major
  double* Gs = fsm + TB * TB;   // Gb_i, column-major: Gs[c + k*TB] = Gb[c][k]
  __shared__ int s_i;
  __shared__ double redt[TB][TB + 1];
  __shared__ double part4[4][TB];
  __shared__ double v[TB];
  __shared__ double cvec[TB];
  const int64_t nblk = (N + TB - 1) / TB;
  if (threadIdx.x == 0) s_i = atomicAdd(ticket, 1);
  __syncthreads();
  const int64_t i = nblk - 1 - s_i;
  const int64_t r0 = i * TB;
  const int nr = (int)((N - r0) < TB ? (N - r0) : TB);
  const int k = threadIdx.x & (TB - 1), cgp = threadIdx.x / TB;
  stage_chain_ops(Bs, Gs, binv + (size_t)i * TB * TB, gb + (size_t)i * TB * TB, i + 1 < nblk);
  const double zi = (threadIdx.x < TB && k < nr) ? z[r0 + k] : 0.0;   // off the chain
  double acc[16];
#pragma unroll
  for (int c = 0; c < 16; c++) acc[c] = 0.0;
  double lv[16], ln[16];
  auto loadL = [&](int64_t q, double* dst) {
    const int64_t row = q * TB + k;
    const bool ok = row < N;
#pragma unroll
    for (int c = 0; c < 16; c++) {
      const int cc = cgp * 16 + c;
      dst[c] = (ok && cc < nr) ? L[row + (r0 + cc) * lda] : 0.0;
    }
  };
  const int64_t qlo = i + 2;   // blocks streamed here (block i+1 goes through Gb_i)
  // x_q is prefetched together with L's block q (one block ahead)
  const unsigned long long ZERO = 0ull;
  unsigned long long xv = ZERO, xn = ZERO;
  if (nblk - 1 >= qlo) {
    loadL(nblk - 1, lv);
    if ((nblk - 1) * TB + k < N) load_values<1>(x + (nblk - 1) * TB + k, &xv);
  }
  for (int64_t q = nblk - 1; q >= qlo; q--) {   // completion order: last block finishes first
    if (q - 1 >= qlo) { loadL(q - 1, ln); load_values<1>(x + (q - 1) * TB + k, &xn); }
    const int64_t row = q * TB + k;
    double xq = 0.0;
    if (row < N) finish_values<1>(x + row, &xv, &xq);
#pragma unroll
    for (int c = 0; c < 16; c++) acc[c] += lv[c] * xq;
#pragma unroll
    for (int c = 0; c < 16; c++) lv[c] = ln[c];
    xv = xn;
  }
  // reduce acc over the 64 rows k: transpose through shared memory (no shuffle chains)
#pragma unroll
  for (int c = 0; c < 16; c++) redt[k][cgp * 16 + c] = acc[c];
  __syncthreads();
  {
    const int c = threadIdx.x & (TB - 1), part = threadIdx.x / TB;   // 4 threads per column, 16 rows each
    double sacc = 0.0;
#pragma unroll
    for (int kk = 0; kk < 16; kk++) sacc += redt[part * 16 + kk][c];
    part4[part][c] = sacc;
  }
  __syncthreads();
  if (threadIdx.x < TB) {
    const int cc = threadIdx.x;
    const double sum = part4[0][cc] + part4[1][cc] + part4[2][cc] + part4[3][cc];
    v[cc] = (cc < nr) ? zi - sum : 0.0;
  }
  __syncthreads();
  // c'_i = Binv^T v : c'[c] = sum_r Binv[r][c] v[r]; thread (c = k, group cgp) sums 16 rows
  double sacc = 0.0;
#pragma unroll
  for (int rr = 0; rr < 16; rr++) {
    const int r = cgp * 16 + rr;
    sacc += Bs[r + k * TB] * v[r];
  }
  part4[cgp][k] = sacc;
  __syncthreads();
  if (threadIdx.x < TB) {
    const int cc = threadIdx.x;
    cvec[cc] = part4[0][cc] + part4[1][cc] + part4[2][cc] + part4[3][cc];
  }
  __syncthreads();
  // the chain step: x_i = c'_i - Gb_i x_{i+1}; thread (c = k, group cgp) sums 16 k's
  double g = 0.0;
  if (i + 1 < nblk) {
    const int64_t rb1 = (i + 1) * TB + cgp * 16;
    double xp[16];
    const int valid = (int)((N - rb1) < 16 ? ((N - rb1) > 0 ? (N - rb1) : 0) : 16);   // ragged last block
    warp_values16(x + rb1, prefetch16(x + rb1, valid), valid, xp);
#pragma unroll
    for (int u = 0; u < 16; u++) g += Gs[k + (cgp * 16 + u) * TB] * xp[u];
  }
  part4[cgp][k] = g;
  __syncthreads();
  if (threadIdx.x < TB) {
    const int cc = threadIdx.x;
    if (cc < nr) publish(&x[r0 + cc], cvec[cc] - ((part4[0][cc] + part4[1][cc]) + (part4[2][cc] + part4[3][cc])));
  }
}

__global__ void k_scatter(int64_t N, const int32_t* __restrict__ piv, const double* __restrict__ y,
                          double* __restrict__ x, BStr z) {
  pdl_wait();
  pdl_trigger();
  piv += blockIdx.y * z.piv; y = bsh(y, z.ws); x += blockIdx.y * z.dxy;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
    x[piv[N + i] & PERM_MASK] = y[i];
}

// dx_s[k] = w[k] * (r_xs[k] - sum_p val[p] * dy[colidx[p]])
__global__ void k_recover(int64_t n_s, const int32_t* __restrict__ rowptr, const int32_t* __restrict__ colidx,
                          const double* __restrict__ val, const double* __restrict__ w,
                          const double* __restrict__ r_xs, const double* __restrict__ dy,
                          double* __restrict__ dx_s, BStr z) {
  pdl_wait();
  pdl_trigger();
  val += blockIdx.y * z.val; w += blockIdx.y * z.w; r_xs += blockIdx.y * z.rxs; dy += blockIdx.y * z.dxy;
  dx_s += blockIdx.y * z.dxs;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n_s; k += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int p = rowptr[k]; p < rowptr[k + 1]; p++) s += val[p] * dy[colidx[p]];
    dx_s[k] = w[k] * (r_xs[k] - s);
  }
}
}  // namespace

extern "C" size_t mds_solve_workspace_size(int64_t N) {
  size_t t = 0;
  carve(nullptr, std::max<int64_t>(N, 1), &t);
  return t;
}

static int solve_launch(const mds_plan* plan, int64_t batch, int64_t N, const double* LD, int64_t ldm,
                        const int32_t* piv, const double* rhs_c, const double* js_val, const double* w,
                        const double* r_xs, double* dxy, double* dx_s, double zero_tol, const void* fwork,
                        int32_t* status, void* work, const BStr& z, cudaStream_t st, bool batched_api = false) {
  const unsigned nb = (unsigned)batch;
  if (N > 0) {
    SWork s = carve(work, N, nullptr);
    const int64_t nblk = (N + TB - 1) / TB;
    const unsigned ge = (unsigned)std::min<int64_t>(mds_cdiv(N, 256), batch > 1 ? 16 : 148 * 8);
    MDS_LAUNCH(PC_SOLVE_GATHER, st, MDS_CUDA_TRY(launch_pdl(k_gather, dim3(ge, nb), dim3(256), 0, st, N, piv, rhs_c, s.b, s.y, s.x, s.tickets, z)));
    if (mds_once_per_device((const void*)k_inv_blocks<true>)) {
      cudaFuncSetAttribute(k_inv_blocks<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, IBSMEM);
      cudaFuncSetAttribute(k_inv_blocks<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, IBSMEM);
      cudaFuncSetAttribute(k_trsv_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, SWSMEM);
      cudaFuncSetAttribute(k_trsv_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, SWSMEM);
    }
    // batched API: one CTA per scenario per sweep (the vector of N doubles in shared memory)
    const bool per_scen = batched_api && (size_t)N * 8 <= (size_t)BSMAX;
    MDS_LAUNCH(PC_SOLVE_FWD, st,
               MDS_CUDA_TRY(launch_pdl(per_scen ? k_inv_blocks<false> : k_inv_blocks<true>, dim3((unsigned)nblk, nb), dim3(256), IBSMEM, st, N, LD, ldm, s.binv,
                                       per_scen ? (double*)nullptr : s.gf, per_scen ? (double*)nullptr : s.gb, z)));
    if (per_scen && mds_once_per_device((const void*)k_bsolve_fwd)) {
      cudaFuncSetAttribute(k_bsolve_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, BSMAX);
      cudaFuncSetAttribute(k_bsolve_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, BSMAX);
    }
    if (per_scen)
      MDS_LAUNCH(PC_SOLVE_FWD, st,
                 MDS_CUDA_TRY(launch_pdl(k_bsolve_fwd, dim3(1, nb), dim3(BST), (size_t)N * 8, st, N, LD, ldm, (const double*)s.b, s.y, (const double*)s.binv, z)));
    else
    MDS_LAUNCH(PC_SOLVE_FWD, st,
               MDS_CUDA_TRY(launch_pdl(k_trsv_fwd, dim3((unsigned)nblk, nb), dim3(ST), SWSMEM, st, N, LD, ldm, s.b, s.y, s.binv, s.gf, s.tickets, z)));
    const double* tolp = (zero_tol < 0.0 && fwork) ? mds_factor_tol_ptr(fwork) : nullptr;
    MDS_LAUNCH(PC_SOLVE_D, st,
               MDS_CUDA_TRY(launch_pdl(k_dsolve, dim3(ge, nb), dim3(256), 0, st, N, LD, ldm, piv, s.y, tolp, zero_tol < 0.0 ? 0.0 : zero_tol, status, z)));
    if (per_scen)
      MDS_LAUNCH(PC_SOLVE_BWD, st,
                 MDS_CUDA_TRY(launch_pdl(k_bsolve_bwd, dim3(1, nb), dim3(BST), (size_t)N * 8, st, N, LD, ldm, (const double*)s.y, s.x, (const double*)s.binv, z)));
    else
    MDS_LAUNCH(PC_SOLVE_BWD, st,
               MDS_CUDA_TRY(launch_pdl(k_trsv_bwd, dim3((unsigned)nblk, nb), dim3(ST), SWSMEM, st, N, LD, ldm, s.y, s.x, s.binv, s.gb, s.tickets + 1, z)));
    MDS_LAUNCH(PC_SOLVE_SCATTER, st, MDS_CUDA_TRY(launch_pdl(k_scatter, dim3(ge, nb), dim3(256), 0, st, N, piv, s.x, dxy, z)));
  }
  if (plan && dx_s) {
    int64_t dims[5];
    mds_plan_dims(plan, dims);
    const int64_t n_s = dims[0], n_d = dims[1];
    if (dims[1] + dims[2] + dims[3] != N) return MDS_ERR_ARG;
    if (n_s > 0) {
      if (!w || !r_xs || (dims[4] > 0 && !js_val)) return MDS_ERR_ARG;
      const unsigned g = (unsigned)std::min<int64_t>(mds_cdiv(n_s, 256), batch > 1 ? 64 : 148 * 16);
      MDS_LAUNCH(PC_RECOVER, st,
                 MDS_CUDA_TRY(launch_pdl(k_recover, dim3(g, nb), dim3(256), 0, st, n_s, mds_plan_rowptr(plan),
                                         mds_plan_colidx(plan), js_val, w, r_xs, dxy + n_d, dx_s, z)));
    }
  }
  return MDS_OK;
}

extern "C" int mds_solve(const mds_plan* plan, int64_t N, const double* LD, int64_t ldm, const int32_t* piv,
                         const double* rhs_c, const double* js_val, const double* w, const double* r_xs,
                         double* dxy, double* dx_s, double zero_tol, const void* fwork, int32_t* status,
                         void* work, size_t work_bytes, void* stream) {
  if (N < 0 || (N > 0 && (!LD || !piv || !rhs_c || !dxy)) || ldm < std::max<int64_t>(N, 1)) return MDS_ERR_ARG;
  if (!work || work_bytes < mds_solve_workspace_size(N)) return MDS_ERR_WORKSPACE;
  const BStr z = {};
  return solve_launch(plan, 1, N, LD, ldm, piv, rhs_c, js_val, w, r_xs, dxy, dx_s, zero_tol, fwork, status, work, z,
                      (cudaStream_t)stream);
}

static size_t solve_ws_stride(int64_t N) { return align_up(mds_solve_workspace_size(N), 256); }

extern "C" size_t mds_solve_batched_workspace_size(int64_t N, int64_t batch) {
  return batch < 1 ? 0 : (size_t)batch * solve_ws_stride(N);
}

extern "C" int mds_solve_batched(const mds_plan* plan, int64_t batch, int64_t N, const double* LD, int64_t ldm,
                                 int64_t str_LD, const int32_t* piv, int64_t str_piv, const double* rhs_c,
                                 int64_t str_rhs, const double* js_val, int64_t str_val, const double* w, int64_t str_w,
                                 const double* r_xs, int64_t str_r, double* dxy, int64_t str_dxy, double* dx_s,
                                 int64_t str_dxs, double zero_tol, const void* fwork, int32_t* status, void* work,
                                 size_t work_bytes, void* stream) {
  if (batch < 0 || N < 0) return MDS_ERR_ARG;
  if (batch == 0) return MDS_OK;
  if (!status) return MDS_ERR_ARG;
  if (N > 0 && (!LD || !piv || !rhs_c || !dxy || ldm < N || str_LD < ldm * N || str_piv < 2 * N ||
                str_rhs < N || str_dxy < N))
    return MDS_ERR_ARG;
  if (!work || work_bytes < mds_solve_batched_workspace_size(N, batch)) return MDS_ERR_WORKSPACE;
  BStr z;
  z.ld = str_LD; z.piv = str_piv; z.rhs = str_rhs; z.dxy = str_dxy; z.val = str_val; z.w = str_w; z.rxs = str_r;
  z.dxs = str_dxs;
  z.ws = solve_ws_stride(N);
  z.fws = mds_factor_ws_stride_bytes(N);
  return solve_launch(plan, batch, N, LD, ldm, piv, rhs_c, js_val, w, r_xs, dxy, dx_s, zero_tol, fwork, status, work,
                      z, (cudaStream_t)stream, true);
}
