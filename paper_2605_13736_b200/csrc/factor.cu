// factor.cu — mds_factor: blocked FP64 Bunch-Kaufman LDL^T with inertia
// (K4; alpha = (1+sqrt 17)/8), designed for sm_100a.
//
// Right-looking, LAPACK-dlasyf-style panels of width NB with a W = L*D work
// panel, followed by a rank-kb trailing update C -= L21 * W21^T that runs on
// the FP64 tensor cores (mma.sync m8n8k4 f64 -> SASS DMMA; there is no FP64
// tcgen05 kind on Blackwell).  Each panel first tries a SPECULATIVE fast path:
//   F1 k_panel_diag   one CTA factors the NB x NB diagonal block without
//                     pivoting (in shared memory),
//   F2 k_panel_trsm   all free SMs form W21 = A21 L11^{-T} (the fully updated
//                     panel columns) and the per-column BK colmax,
//   F4 k_panel_slow   accepts the longest prefix of columns that pass BK's
//                     1x1-no-interchange test |d_k| >= alpha*colmax_k (the test
//                     BK itself applies to exactly these numbers),
// and recomputes the columns after the first failing one with the exact
// sequential BK panel (dlasyf semantics: rowmax, 1x1 / 2x2 / interchange).
// The panel's D + L live in a side buffer Lb until k_panel_store copies them
// into M (off the critical path, on the look-ahead stream).
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
#include <cuda.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <map>
#include <mutex>
#include <vector>

#include "anorm.cuh"
#include "common.cuh"

namespace cg = cooperative_groups;

namespace {
constexpr int NB = 64;              // panel width
constexpr int WCOLS = NB + 1;       // W work panel columns (+1 for the 2x2 candidate)
constexpr int XT = 512;             // threads per CTA of the multi-CTA exact panel (k_panel_exact)
constexpr int XMAXG = 256;          // its maximum grid
constexpr int XROWS = XT / 4;       // rows per CTA pass (a quad of threads per row)
constexpr int XLS_MAX = 200 * 1024; // k_panel_exact's shared-memory copy of its L rows (else read from L2)
constexpr double ALPHA_BK = 0.64038820320220756872767623199676;  // (1+sqrt(17))/8

struct FCtl {
  int k0;          // first column of the current panel
  int kb;          // columns finished in the current panel
  int nbp;         // width of the current panel's diagonal block
  int npanel;      // panels started
  int nswap;       // interchanges performed (kp != kk)
  int abort;       // non-finite input: nothing is factored
  unsigned xready; // q+1 once panel q's F1 has published X, d and the in-block colmax
  int nexact;     // columns decided by the exact (dlasyf) BK steps rather than the accepted prefix
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
  char* nparts;       // ||M||_inf partials (anorm.cuh), parts_bytes(N)
  double* Lblk;       // [NB*NB]
  double* W;          // [ldw * WCOLS]  W panel of the current panel (host picks W0/W1 by panel parity)
  double* W1;         // second W buffer (look-ahead: panel p+1 is formed while p's update still reads W)
  double* Lb;         // [ldw * WCOLS]  the panel's D + L columns (speculative, fixed up by k_panel_slow);
  double* Lb1;        //   copied into M by k_panel_store; double-buffered like W
  int2* pinfo;        // [N+2] per-panel (k0, kb), written by k_panel_slow, read by the updates
  unsigned long long* ucount;   // [3(N+2)] per-panel tile counters: [3q] rest/full update, [3q+1] next-panel
                                //   update, [3q+2] F2 tiles of panel q (claimed by k_panel_trsm and k_update_tma<3, true>)
  unsigned* t1flag;             // [2(N/64+4)] p+1 once panel p's update of tile (row BI, column b0+c) has landed
  unsigned* xbar;               // [N/32+8] per-panel grid-barrier counters of k_panel_exact
  ArgMax* xpart;                // [2 banks][XMAXG] its per-CTA argmax partials (bank = barrier parity)
  double* xpay;                 // [2 banks][XMAXG][2] per-CTA payloads of those exchanges (W values of one owned row)
  const double* Wprev;          // the previous panel's W / Lb (the other parity buffers), for the
  const double* Lbprev;         //   deferred update of this panel's columns
  int fuse;           // 1: this panel's columns still lack the previous panel's update (look-ahead)
  int pidx;           // panel index of this launch (host loop counter)
  int64_t ldw;
  // batched factorization (mds_factor_batched): scenario s = blockIdx.y (z for k_panel_store)
  // owns the workspace at + s * bws bytes, M at + s * bms elements, piv at + s * bps
  size_t bws;
  int64_t bms, bps;
  // emulated-FP64 update (ozaki.cuh): int8 slices [8][N][64] of the panel's L and W, row exponents
  int8_t* ozL;
  int8_t* ozW;
  int* ozeL;
  int* ozeW;
};

template <typename T>
__device__ __forceinline__ void shp(T*& p, size_t o) { p = reinterpret_cast<T*>(reinterpret_cast<uintptr_t>(p) + o); }
// this scenario's view of a batched factorization (no-op for s = 0 / single system):
// workspace pointers of f, and the caller's M (and piv) pointers
__device__ __forceinline__ void bsel_ws(FWork& f, int64_t s) {
  if (s == 0) return;
  const size_t o = (size_t)s * f.bws;
  shp(f.ctl, o); shp(f.panel_start, o); shp(f.sw, o); shp(f.bt, o); shp(f.rho, o); shp(f.rhoinv, o);
  shp(f.nparts, o); shp(f.Lblk, o); shp(f.W, o); shp(f.W1, o); shp(f.Lb, o); shp(f.Lb1, o); shp(f.pinfo, o);
  shp(f.ucount, o); shp(f.t1flag, o); shp(f.xbar, o); shp(f.xpart, o); shp(f.xpay, o); shp(f.Wprev, o);
  shp(f.Lbprev, o); shp(f.ozL, o); shp(f.ozW, o); shp(f.ozeL, o); shp(f.ozeW, o);
}

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
  f.nparts = take(anorm::parts_bytes(N));
  f.Lblk = reinterpret_cast<double*>(take(sizeof(double) * NB * NB));
  f.ldw = align_up(std::max<int64_t>(N, 1), 8);
  f.W = reinterpret_cast<double*>(take(sizeof(double) * f.ldw * WCOLS));
  f.W1 = reinterpret_cast<double*>(take(sizeof(double) * f.ldw * WCOLS));
  f.Lb = reinterpret_cast<double*>(take(sizeof(double) * f.ldw * WCOLS));
  f.Lb1 = reinterpret_cast<double*>(take(sizeof(double) * f.ldw * WCOLS));
  f.pinfo = reinterpret_cast<int2*>(take(sizeof(int2) * (N + 2)));
  f.ucount = reinterpret_cast<unsigned long long*>(take(sizeof(unsigned long long) * 3 * (N + 2)));
  f.t1flag = reinterpret_cast<unsigned*>(take(sizeof(unsigned) * 2 * (N / 64 + 4)));
  f.xbar = reinterpret_cast<unsigned*>(take(sizeof(unsigned) * (N / 32 + 8)));
  f.xpart = reinterpret_cast<ArgMax*>(take(sizeof(ArgMax) * 2 * XMAXG));
  f.xpay = reinterpret_cast<double*>(take(sizeof(double) * 2 * XMAXG * 2));
  f.ozL = reinterpret_cast<int8_t*>(take((size_t)8 * N * 64));
  f.ozW = reinterpret_cast<int8_t*>(take((size_t)8 * N * 64));
  f.ozeL = reinterpret_cast<int*>(take(sizeof(int) * N));
  f.ozeW = reinterpret_cast<int*>(take(sizeof(int) * N));
  f.Wprev = f.W1;
  f.Lbprev = f.Lb1;
  f.fuse = 0;
  f.pidx = 0;
  f.bws = 0;
  f.bms = 0;
  f.bps = 0;
  if (total) *total = off;
  return f;
}

// reciprocal for the pivot multipliers: MUFU seed + 2 Newton steps (off the
// correctly-rounded slow path; the oracle's 1/d differs by <= 1 ulp)
__device__ __forceinline__ double fast_rcp(double d) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  const double e = fma(-d, r, 1.0);          // r (1 + e + e^2): 3 dependent FP64 ops after the seed
  return fma(r, fma(e, e, e), r);
}
__device__ __forceinline__ unsigned long long dbits(double v) { return (unsigned long long)__double_as_longlong(v); }
__device__ __forceinline__ double bitsd(unsigned long long b) { return __longlong_as_double((long long)b); }

// ---------------------------------------------------------------------------
// zero the per-call control state (one kernel instead of several memsets, so
// the launch chain stays programmatic-dependent-launch friendly)
__global__ void k_factor_init(int64_t N, FWork f, double zero_tol, const double* anorm, int32_t* status,
                              const int32_t* active) {
  {   // batched: scenario blockIdx.y
    bsel_ws(f, blockIdx.y);
    if (status) status += blockIdx.y;
    if (anorm) anorm += blockIdx.y;
  }
  pdl_wait();
  pdl_trigger();
  if (active && !active[blockIdx.y]) {
    // scenario not re-factored this call: keep its factorization, tolerance and counters;
    // abort = 2 makes every later kernel of this call skip it (finalize leaves its outputs alone)
    if (blockIdx.x == 0 && threadIdx.x == 0) f.ctl->abort = 2;
    return;
  }
  const int64_t gtid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t gth = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = gtid; i < N; i += gth) { f.sw[i] = -1; f.bt[i] = 0; }
  for (int64_t i = gtid; i < 3 * (N + 2); i += gth) f.ucount[i] = 0ull;
  for (int64_t i = gtid; i < 2 * (N / 64 + 4); i += gth) f.t1flag[i] = 0u;
  for (int64_t i = gtid; i < N / 32 + 8; i += gth) f.xbar[i] = 0u;
  if (gtid < 4) anorm::parts_at(f.nparts, N).ctr[gtid] = 0u;
  if (blockIdx.x == 0) {
    int* c = reinterpret_cast<int*>(f.ctl);
    for (int i = threadIdx.x; i < (int)(sizeof(FCtl) / sizeof(int)); i += blockDim.x) c[i] = 0;
    __syncthreads();
    if (threadIdx.x == 0) {
      f.ctl->tol = zero_tol;
      if (anorm) {   // ||M||_inf provided by the condensation (a3 fused into a2)
        const double a = *anorm;
        f.ctl->anorm = a;
        if (!isfinite(a)) {   // NaN marks a non-finite M (anorm.cuh)
          f.ctl->abort = 1;
          mds_set_status(status, MDS_ERR_NONFINITE);
        } else if (zero_tol < 0.0) {
          f.ctl->tol = (double)N * 2.220446049250313e-16 * a;
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Panel fast path.
//   F1 k_panel_diag (1 CTA): apply the previous panel's rank-kb update to the
//       64x64 diagonal block (with look-ahead the trailing update of panel p
//       never touches it, so F1 starts right after panel p's exact step),
//       unpivoted LDL^T of the block in shared memory (16-column blocks:
//       warp-register panels + register-blocked rank-16 trailing updates),
//       L11^{-1} by blocked inversion.  Leaves X = L11^{-T} (row-major
//       [t][j]) in Lblk, W11 / D + L11 in W / Lb, d and the in-block colmax.
//   F2 k_panel_trsm (all free SMs): W21 = A21 X (DMMA), speculative
//       L21 = W21 D^{-1}, per-column colmax.
#ifdef MDS_F1_TIMING
__device__ long long g_f1t[8];
#define F1T(i) do { __syncthreads(); if (threadIdx.x == 0) g_f1t[i] = clock64(); } while (0)
#else
#define F1T(i) do { } while (0)
#endif
#ifdef MDS_F1_TRACE   // tools/factor_trace.cu: per-panel F1 wall time and SM cycles
__device__ unsigned long long g_f1trace[4096][8];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define F1TRACE(k) do { if (threadIdx.x == 0 && f.pidx < 4096) { g_f1trace[f.pidx][2 * (k)] = gtimer(); g_f1trace[f.pidx][2 * (k) + 1] = clock64(); } } while (0)
// [0] U start (min), [1] U end (max), [2] F2 tiles done in U, [3] trsm start, [4] trsm end, [5] trsm tiles
__device__ unsigned long long g_utrace[4096][6];
__device__ unsigned long long g_usm[512][160][2];   // per panel, per SM: U CTA start / end
__device__ unsigned g_f1sm[4096];
__device__ __forceinline__ unsigned smid() { unsigned r; asm volatile("mov.u32 %0, %smid;" : "=r"(r)); return r; }
#define USM_START(p) do { if ((p) < 512) atomicMin(&g_usm[p][smid()][0], gtimer()); } while (0)
#define USM_END(p) do { if ((p) < 512) atomicMax(&g_usm[p][smid()][1], gtimer()); } while (0)
#define F1SM() do { if (threadIdx.x == 0 && f.pidx < 4096) g_f1sm[f.pidx] = smid(); } while (0)
#define UTRACE_MIN(p, k) atomicMin(&g_utrace[p][k], gtimer())
#define UTRACE_MAX(p, k) atomicMax(&g_utrace[p][k], gtimer())
#define UTRACE_ADD(p, k) atomicAdd(&g_utrace[p][k], 1ull)
__device__ unsigned long long g_f4trace[4096][2];   // k_panel_exact: [0] first CTA past pdl_wait (min), [1] last exit (max)
// per-phase cycles of CTA 0 of k_panel_exact, summed over all exact columns (tools/exact_trace.cu)
__device__ unsigned long long g_xph[10];
#define XPH_DECL unsigned long long xph_t = clock64()
#define XPH(i) do { if (threadIdx.x == 0 && blockIdx.x == 0) { const unsigned long long t_ = clock64(); atomicAdd(&g_xph[i], t_ - xph_t); xph_t = t_; } } while (0)
#define XPH_COUNT atomicAdd(&g_xph[9], 1ull)
#define F4TRACE_MIN(p) do { if (threadIdx.x == 0 && (p) < 4096) atomicMin(&g_f4trace[p][0], gtimer()); } while (0)
#define F4TRACE_MAX(p) do { if (threadIdx.x == 0 && (p) < 4096) atomicMax(&g_f4trace[p][1], gtimer()); } while (0)
#else
#define F4TRACE_MIN(p) do { } while (0)
#define F4TRACE_MAX(p) do { } while (0)
#define XPH_DECL do { } while (0)
#define XPH(i) do { } while (0)
#define XPH_COUNT do { } while (0)
#define UTRACE_MIN(p, k) do { } while (0)
#define UTRACE_MAX(p, k) do { } while (0)
#define UTRACE_ADD(p, k) do { } while (0)
#define USM_START(p) do { } while (0)
#define USM_END(p) do { } while (0)
#define F1SM() do { } while (0)
#define F1TRACE(k) do { } while (0)
#endif
constexpr int F1S = NB + 1;                     // F1 smem column stride
constexpr int UT = 64;                          // DMMA tile edge
constexpr int US = UT + 4;                      // F2 smem row stride (conflict-free fragment loads)
static_assert(UT == NB, "X staging assumes square 64x64 tiles");
// X = L11^{-T} (row-major [t][j], NB x NB in f.Lblk) into shared memory at row
// stride US, with up to 16 loads of a thread in flight before its stores (a
// load-store loop waits one round trip per element)
template <int NT, bool CG>
__device__ __forceinline__ void stage_x(double* dst, const double* __restrict__ src, int tid) {
  constexpr int PER = NB * NB / NT;
  constexpr int H = PER > 16 ? 16 : PER;
#pragma unroll
  for (int h = 0; h < PER; h += H) {
    double v[H];
#pragma unroll
    for (int u = 0; u < H; u++) {
      const int idx = tid + (h + u) * NT;
      v[u] = CG ? __ldcg(&src[idx]) : src[idx];
    }
#pragma unroll
    for (int u = 0; u < H; u++) {
      const int idx = tid + (h + u) * NT;
      dst[(idx >> 6) * US + (idx & (NB - 1))] = v[u];
    }
  }
}
constexpr int PF_BUF = NB * US;                 // doubles per shared buffer (>= NB * F1S)
constexpr int F1SMEM = (3 * PF_BUF + NB) * 8;   // 3 buffers + 1/d

// FP64 tensor-core fragment op: mma.sync m8n8k4 f64 (SASS DMMA.8x8x4).
// a0 = A[g][q], b0 = B[q][g], {c0,c1} = C[g][2q], C[g][2q+1]  (g = lane>>2, q = lane&3)
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
// plain (non-warp-aggregated) 64-bit fetch-add: the compiler's atomicAdd from a single
// lane becomes a match/popc/shuffle sequence that consumes the result at once,
// which would serialise the producer's one-ahead tile claim
__device__ __forceinline__ unsigned long long atom_add_u64(unsigned long long* p, unsigned long long v) {
  unsigned long long r;
  asm volatile("atom.global.add.u64 %0, [%1], %2;\n" : "=l"(r) : "l"(p), "l"(v) : "memory");
  return r;
}
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
// first column of this launch's panel: end of the previous panel (written by its k_panel_slow)
__device__ __forceinline__ int64_t panel_k0(const FWork& f) {
  if (f.pidx == 0) return 0;
  const int2 pp = f.pinfo[f.pidx - 1];
  return (int64_t)pp.x + pp.y;
}

// One warp factors a 16-column panel (rows cb..63) held in registers: lane
// owns rows cb+lane (+32); pivots and column values broadcast by shuffles.
// The block is padded with the identity beyond nbp, so every block has 16
// columns and nothing is predicated: entries above the diagonal are updated
// with garbage that is never read (only the lower triangle, the diagonal and
// the multipliers below it feed later steps).
template <int SLOTS>
__device__ __forceinline__ void f1_panel(double* As, double* Lm, double* rcp, int cb, int lane) {
  // fully unrolled (column index compile-time, so pv stays in registers and the
  // triangular loop does only the live updates); no per-element predicates, so
  // the straight-line code stays small enough for the instruction cache
  double pv[SLOTS][16];
  int rr[SLOTS];
#pragma unroll
  for (int sl = 0; sl < SLOTS; sl++) {
    rr[sl] = cb + 32 * sl + lane;
#pragma unroll
    for (int c = 0; c < 16; c++) pv[sl][c] = (rr[sl] < NB) ? As[(cb + c) * F1S + rr[sl]] : 0.0;
  }
#pragma unroll
  for (int jj = 0; jj < 16; jj++) {
    const int j = cb + jj;
    const double d = __shfl_sync(0xffffffffu, pv[0][jj], jj);
    const double rd = fast_rcp(d);               // branch-free (keeps the shuffles convergent)
    const double r1 = (d != 0.0) ? rd : 0.0;
    double l[SLOTS];
#pragma unroll
    for (int sl = 0; sl < SLOTS; sl++) l[sl] = pv[sl][jj] * r1;
#pragma unroll
    for (int c = jj + 1; c < 16; c++) {
      const double v = __shfl_sync(0xffffffffu, pv[0][jj], c);   // A(cb+c, j)
#pragma unroll
      for (int sl = 0; sl < SLOTS; sl++) pv[sl][c] -= l[sl] * v;
    }
    if (lane == 0) rcp[j] = r1;
#pragma unroll
    for (int sl = 0; sl < SLOTS; sl++) {
      if (SLOTS == 1 || rr[sl] < NB) Lm[j * F1S + rr[sl]] = l[sl];         // multipliers of column j
      if (rr[sl] < NB && rr[sl] >= j) As[j * F1S + rr[sl]] = pv[sl][jj];   // column j is final
    }
  }
}

__device__ __forceinline__ void f1_body(int64_t N, double* __restrict__ A, int64_t lda, const FWork& f, int64_t k0,
                                        int nbp, bool fprev, double* sm) {
  FCtl* ctl = f.ctl;
  double* As = sm;                   // As[c*F1S + r] : the block, updated in place (lower)
  double* Lm = sm + PF_BUF;          // Lm[c*F1S + r] = L[r][c] (unit lower multipliers, r > c); staging: Lprev
  double* Li = sm + 2 * PF_BUF;      // Li[c*F1S + r] = Linv[r][c];                              staging: Wprev
  double* Tm = As;                   // temp GEMM block of the inversion (As is dead by then)
  double* rcp = sm + 3 * PF_BUF;     // 1/d_j (0 for an exactly zero pivot)
  const int tid = threadIdx.x;
  const int64_t ldw = f.ldw;
  F1T(0);
  F1TRACE(0);
  F1SM();
  {
    // all loads of a thread in flight at once
    double v[16];
    const int r = tid & (NB - 1), c0 = tid >> 6;
    const double* src = A + (k0 + r) + (k0 + c0) * lda;
#pragma unroll
    for (int u = 0; u < 16; u++) {
      const int c = c0 + 4 * u;
      v[u] = (r >= c && r < nbp && c < nbp) ? src[(int64_t)(4 * u) * lda] : (r == c ? 1.0 : 0.0);   // identity pad
    }
    if (fprev) {
      double lp[16];
#pragma unroll
      for (int u = 0; u < 16; u++) lp[u] = (r < nbp) ? f.Lbprev[(k0 + r) + (c0 + 4 * u) * ldw] : 0.0;
#pragma unroll
      for (int u = 0; u < 16; u++) As[(c0 + 4 * u) * F1S + r] = v[u];
#pragma unroll
      for (int u = 0; u < 16; u++) v[u] = (r < nbp) ? f.Wprev[(k0 + r) + (c0 + 4 * u) * ldw] : 0.0;
#pragma unroll
      for (int u = 0; u < 16; u++) Lm[(c0 + 4 * u) * F1S + r] = lp[u];
#pragma unroll
      for (int u = 0; u < 16; u++) Li[(c0 + 4 * u) * F1S + r] = v[u];
    } else {
#pragma unroll
      for (int u = 0; u < 16; u++) As[(c0 + 4 * u) * F1S + r] = v[u];
    }
  }
  __syncthreads();
  if (fprev) {
    // deferred update of the previous panel on the FP64 tensor cores:
    // A11 -= Lprev(k0:k0+64, :) Wprev(k0:k0+64, :)^T; warp w owns rows 32(w&1).., cols 16(w>>1)..
    const int warp = tid >> 5, lane = tid & 31, g = lane >> 2, q = lane & 3;
    const int wm = (warp & 1) * 32, wn = (warp >> 1) * 16;
    double acc[4][2][2];
#pragma unroll
    for (int a = 0; a < 4; a++)
#pragma unroll
      for (int b = 0; b < 2; b++) acc[a][b][0] = acc[a][b][1] = 0.0;
    if (wm + 31 >= wn) {   // warps entirely above the diagonal have nothing to do
#pragma unroll 4
      for (int t0 = 0; t0 < NB; t0 += 4) {
        double av[4], bv[2];
#pragma unroll
        for (int a = 0; a < 4; a++) av[a] = Lm[(t0 + q) * F1S + wm + 8 * a + g];
#pragma unroll
        for (int b = 0; b < 2; b++) bv[b] = Li[(t0 + q) * F1S + wn + 8 * b + g];
#pragma unroll
        for (int a = 0; a < 4; a++)
#pragma unroll
          for (int b = 0; b < 2; b++) dmma(acc[a][b][0], acc[a][b][1], av[a], bv[b]);
      }
    }
#pragma unroll
    for (int a = 0; a < 4; a++)
#pragma unroll
      for (int b = 0; b < 2; b++)
#pragma unroll
        for (int e = 0; e < 2; e++) {
          const int r = wm + 8 * a + g, c = wn + 8 * b + 2 * q + e;
          if (r >= c && r < nbp && c < nbp) {
            const double nv = As[c * F1S + r] - acc[a][b][e];
            As[c * F1S + r] = nv;
            A[(k0 + r) + (k0 + c) * lda] = nv;   // updated values for the exact path
          }
        }
    __syncthreads();
  }
  F1T(1);
  F1TRACE(1);
  // ---- factorization, 16-column blocks.  Panel (rows cb.., 16 columns) by warp 0
  // in registers (lane owns rows cb+lane, cb+32+lane; broadcasts by shuffles,
  // no block barriers); the trailing part by all threads, register-blocked.
  const int warp = tid >> 5, lane = tid & 31;
#pragma unroll 1
  for (int cb = 0; cb < NB; cb += 16) {
    const int ce = cb + 16;   // (the identity pad makes every block 16 wide)
    if (warp == 0) {
      if (cb < 32) f1_panel<2>(As, Lm, rcp, cb, lane);
      else f1_panel<1>(As, Lm, rcp, cb, lane);
    }
    __syncthreads();
    if (cb == 0) F1T(6);
    // rank-(ce-cb) update of the trailing part (rows/cols >= ce, lower): 16x16 threads x 3x3 blocks
    if (ce < nbp) {
      const int tr = tid & 15, tc = tid >> 4;
      double acc[3][3];
#pragma unroll
      for (int a = 0; a < 3; a++)
#pragma unroll
        for (int b = 0; b < 3; b++) {
          const int r = ce + tr + 16 * a, c = ce + tc + 16 * b;
          acc[a][b] = (r < nbp && c < nbp && r >= c) ? As[c * F1S + r] : 0.0;
        }
#pragma unroll 4
      for (int t = 0; t < 16; t++) {
        double lr[3], wc[3];
#pragma unroll
        for (int a = 0; a < 3; a++) {
          const int r = ce + tr + 16 * a;
          lr[a] = (r < NB) ? Lm[(cb + t) * F1S + r] : 0.0;
        }
#pragma unroll
        for (int b = 0; b < 3; b++) {
          const int c = ce + tc + 16 * b;
          wc[b] = (c < NB) ? As[(cb + t) * F1S + c] : 0.0;
        }
#pragma unroll
        for (int a = 0; a < 3; a++)
#pragma unroll
          for (int b = 0; b < 3; b++) acc[a][b] -= lr[a] * wc[b];
      }
#pragma unroll
      for (int a = 0; a < 3; a++)
#pragma unroll
        for (int b = 0; b < 3; b++) {
          const int r = ce + tr + 16 * a, c = ce + tc + 16 * b;
          if (r < nbp && c < nbp && r >= c) As[c * F1S + r] = acc[a][b];
        }
    }
    __syncthreads();
    if (cb == 0) F1T(5);
  }
  F1T(2);
  F1TRACE(2);
  // ---- outputs that need As / Lm: W11 (updated, unscaled), D + L11 into Lb, d, in-block colmax
  {
    const int j = tid & (NB - 1), t0 = tid >> 6;
    double* Wg = f.W + k0;
#pragma unroll
    for (int u = 0; u < 16; u++) {
      const int t = t0 + 4 * u;
      if (j >= t && j < nbp && t < nbp) {
        Wg[j + t * ldw] = As[t * F1S + j];                                           // W11 (r=j, col=t)
        f.Lb[(k0 + j) + t * ldw] = (j == t) ? As[t * F1S + t] : Lm[t * F1S + j];     // D / L11
      }
    }
  }
  {
    // in-block colmax of column j: 4 threads per column, shuffle-reduced
    const int j = tid >> 2, part = tid & 3;
    double cm = 0.0;
    for (int r = j + 1 + part; r < nbp; r += 4) cm = fmax(cm, fabs(As[j * F1S + r]));
    cm = fmax(cm, __shfl_xor_sync(0xffffffffu, cm, 1));
    cm = fmax(cm, __shfl_xor_sync(0xffffffffu, cm, 2));
    if (part == 0 && j < nbp) { ctl->colmax[j] = dbits(cm); ctl->d[j] = As[j * F1S + j]; }
  }
  __syncthreads();   // As becomes the inversion's temp block
  // ---- L11^{-1}: Lunit[r][c] = As[c][r] * rcp[c] (r > c)
  // (1) diagonal 16x16 blocks: warp w<4 inverts block w; lane c<16 owns column c.
  //     Right-looking: once x_k is final, s_r += L[r][k] x_k for all r > k (independent FMAs),
  //     so the dependent chain is one FMA per row.
  //     (the strictly upper blocks of Li are never read; off-diagonal lower blocks are written in (2))
  if (warp < 4 && lane < 16) {
    const int o = warp * 16, c = lane;
    double x[16];
#pragma unroll
    for (int r = 0; r < 16; r++) x[r] = (r == c) ? 1.0 : 0.0;
#pragma unroll
    for (int k = 0; k < 15; k++) {
      const double xk = x[k];
#pragma unroll
      for (int r = k + 1; r < 16; r++) {
        x[r] = fma(-Lm[(o + k) * F1S + o + r], xk, x[r]);   // (x[k] = 0 for k < c: rows <= c stay e_c)
      }
    }
#pragma unroll
    for (int r = 0; r < 16; r++) Li[(o + c) * F1S + o + r] = (o + r < nbp && o + c < nbp) ? x[r] : 0.0;
  }
  __syncthreads();
  F1T(7);
  // (2) off-diagonal blocks by distance dd: Linv_ij = -Linv_ii * sum_{k=j}^{i-1} L_ik Linv_kj
  //     (4 independent partial sums per dot, all blocks of a distance interleaved)
  const int er = tid & 15, ec = tid >> 4;   // element (er, ec) of a 16x16 block
#pragma unroll
  for (int dd = 1; dd < 4; dd++) {
    double tv[3];
#pragma unroll
    for (int bj = 0; bj < 3; bj++) {
      if (bj + dd < 4) {
        const int bi = bj + dd;
        double p0 = 0.0, p1 = 0.0, p2 = 0.0, p3 = 0.0;
#pragma unroll
        for (int kb2 = bj; kb2 < bi; kb2++)
#pragma unroll
          for (int k = 0; k < 16; k += 4) {
            const int kk = kb2 * 16 + k;
            const double* lr = Lm + bi * 16 + er;
            const double* lc = Li + (bj * 16 + ec) * F1S;
            p0 = fma(lr[(kk + 0) * F1S], lc[kk + 0], p0);
            p1 = fma(lr[(kk + 1) * F1S], lc[kk + 1], p1);
            p2 = fma(lr[(kk + 2) * F1S], lc[kk + 2], p2);
            p3 = fma(lr[(kk + 3) * F1S], lc[kk + 3], p3);
          }
        tv[bj] = (p0 + p1) + (p2 + p3);
      }
    }
#pragma unroll
    for (int bj = 0; bj < 3; bj++)
      if (bj + dd < 4) Tm[(bj * 16 + ec) * F1S + (bj + dd) * 16 + er] = tv[bj];
    __syncthreads();
#pragma unroll
    for (int bj = 0; bj < 3; bj++) {
      if (bj + dd < 4) {
        const int bi = bj + dd;
        double p0 = 0.0, p1 = 0.0, p2 = 0.0, p3 = 0.0;
        const double* li = Li + bi * 16 + er;
        const double* tc = Tm + (bj * 16 + ec) * F1S + bi * 16;
#pragma unroll
        for (int k = 0; k < 16; k += 4) {
          p0 = fma(li[(bi * 16 + k + 0) * F1S], tc[k + 0], p0);
          p1 = fma(li[(bi * 16 + k + 1) * F1S], tc[k + 1], p1);
          p2 = fma(li[(bi * 16 + k + 2) * F1S], tc[k + 2], p2);
          p3 = fma(li[(bi * 16 + k + 3) * F1S], tc[k + 3], p3);
        }
        tv[bj] = (p0 + p1) + (p2 + p3);
      }
    }
#pragma unroll
    for (int bj = 0; bj < 3; bj++) {
      if (bj + dd < 4) {
        const int r = (bj + dd) * 16 + er, c = bj * 16 + ec;
        Li[c * F1S + r] = (r < nbp && c < nbp) ? -tv[bj] : 0.0;
      }
    }
    __syncthreads();
  }
  F1T(3);
  // ---- X[t][j] = Linv[j][t] (row-major, 0 above the diagonal)
  {
    const int j = tid & (NB - 1), t0 = tid >> 6;
#pragma unroll
    for (int u = 0; u < 16; u++) {
      const int t = t0 + 4 * u;
      f.Lblk[t * NB + j] = (j >= t) ? Li[t * F1S + j] : 0.0;
    }
  }
  if (tid == 0) {
    ctl->k0 = (int)k0;
    ctl->kb = 0;
    ctl->nbp = nbp;
    f.panel_start[f.pidx] = (int)k0;
    ctl->npanel = f.pidx + 1;
  }
  __syncthreads();
  if (tid == 0) {   // publish X / d / colmax to the F2 tiles run inside the concurrent trailing update
    // (st.release.gpu is cumulative over the CTA's writes ordered before it by the barrier)
    st_release_u32(&ctl->xready, (unsigned)(f.pidx + 1));
  }
  F1T(4);
  F1TRACE(3);
}

__global__ void __launch_bounds__(256) k_panel_diag(int64_t N, double* __restrict__ A, int64_t lda, FWork f) {
  bsel_ws(f, blockIdx.y);
  A += blockIdx.y * f.bms;
  pdl_wait();
  FCtl* ctl = f.ctl;
  if (ctl->abort) return;
  const int64_t k0 = panel_k0(f);
  if (k0 >= N) {
    if (threadIdx.x == 0) { ctl->k0 = (int)N; ctl->kb = 0; ctl->nbp = 0; }
    return;
  }
  extern __shared__ double sm[];
  f1_body(N, A, lda, f, k0, (int)((N - k0) < NB ? (N - k0) : NB), f.fuse && f.pidx > 0, sm);
}

// Tail-phase panel (the trailing update is short, SMs are free): one launch.
// The first CTA to arrive (ticket 0) takes the F1 role; every other CTA takes
// 64-row tiles below the diagonal block and, while F1 runs, applies the
// previous panel's deferred update to them (A21 -= Lprev Wprev^T, DMMA;
// written back to M for the exact path), then waits for F1's X (the F1 role
// never waits on anything, so this cannot deadlock) and forms W21 = A21 X,
// L21 and colmax.  The concurrent trailing update skips these columns.
__device__ __forceinline__ void f2_role(int64_t N, double* __restrict__ A, int64_t lda, const FWork& f, int64_t k0,
                                        int nbp, bool fprev, int role, int nrole, double* sm) {
  FCtl* ctl = f.ctl;
  const int64_t rb = k0 + nbp;
  const int64_t rbase = (rb / UT) * UT;
  const int64_t ntile = (N > rb) ? (N + UT - 1) / UT - rb / UT : 0;
  int64_t tix = role - 1;
  if (tix >= ntile) return;
  double* S0 = sm;                   // Lprev tile [t][row], then A21 (updated) [col][row]
  double* S1 = sm + PF_BUF;          // Wprev rows of the block [t][c]
  double* S2 = sm + 2 * PF_BUF;      // X [t][j]
  double* r1s = sm + 3 * PF_BUF;
  __shared__ double cmx[8][16];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, q = lane & 3;
  const int wm = (warp & 1) * 32, wn = (warp >> 1) * 16;
  const int64_t ldw = f.ldw;
  if (fprev)
    for (int idx = tid; idx < NB * NB; idx += 256) {
      const int i = idx & (NB - 1), t = idx >> 6;
      S1[t * US + i] = (i < nbp) ? f.Wprev[(k0 + i) + t * ldw] : 0.0;
    }
  double cm[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
  bool haveX = false;
  for (; tix < ntile; tix += nrole) {
    const int64_t R0 = rbase + tix * UT;
    if (fprev) {
      for (int idx = tid; idx < NB * UT; idx += 256) {
        const int i = idx & (UT - 1), t = idx >> 6;
        S0[t * US + i] = (R0 + i < N && R0 + i >= rb) ? f.Lbprev[(R0 + i) + t * ldw] : 0.0;
      }
      double acc[4][2][2];
#pragma unroll
      for (int a = 0; a < 4; a++)
#pragma unroll
        for (int b = 0; b < 2; b++)
#pragma unroll
          for (int e = 0; e < 2; e++) {
            const int64_t row = R0 + wm + 8 * a + g;
            const int col = wn + 8 * b + 2 * q + e;
            acc[a][b][e] = (row < N && row >= rb && col < nbp) ? A[row + (k0 + col) * lda] : 0.0;
          }
      __syncthreads();
#pragma unroll 4
      for (int t0 = 0; t0 < NB; t0 += 4) {
        double av[4], bv[2];
#pragma unroll
        for (int a = 0; a < 4; a++) av[a] = -S0[(t0 + q) * US + wm + 8 * a + g];
#pragma unroll
        for (int b = 0; b < 2; b++) bv[b] = S1[(t0 + q) * US + wn + 8 * b + g];
#pragma unroll
        for (int a = 0; a < 4; a++)
#pragma unroll
          for (int b = 0; b < 2; b++) dmma(acc[a][b][0], acc[a][b][1], av[a], bv[b]);
      }
      __syncthreads();   // every warp is done with the Lprev tile
#pragma unroll
      for (int a = 0; a < 4; a++)
#pragma unroll
        for (int b = 0; b < 2; b++)
#pragma unroll
          for (int e = 0; e < 2; e++) {
            const int r = wm + 8 * a + g, c = wn + 8 * b + 2 * q + e;
            S0[c * US + r] = acc[a][b][e];
            if (R0 + r < N && R0 + r >= rb && c < nbp) A[(R0 + r) + (k0 + c) * lda] = acc[a][b][e];
          }
    } else {
      for (int idx = tid; idx < NB * UT; idx += 256) {
        const int i = idx & (UT - 1), t = idx >> 6;
        S0[t * US + i] = (t < nbp && R0 + i < N && R0 + i >= rb) ? A[(R0 + i) + (k0 + t) * lda] : 0.0;
      }
    }
    if (!haveX) {
      if (tid == 0) {
        while (ld_acquire_u32(&ctl->xready) < (unsigned)(f.pidx + 1)) __nanosleep(32);
      }
      __syncthreads();
      stage_x<256, true>(S2, f.Lblk, tid);
      if (tid < NB) {
        const double d = (tid < nbp) ? __ldcg(&ctl->d[tid]) : 0.0;
        const double rd = fast_rcp(d);
        r1s[tid] = (d != 0.0) ? rd : 0.0;
      }
      haveX = true;
    }
    __syncthreads();
    double acc[4][2][2];
#pragma unroll
    for (int a = 0; a < 4; a++)
#pragma unroll
      for (int b = 0; b < 2; b++) acc[a][b][0] = acc[a][b][1] = 0.0;
#pragma unroll 4
    for (int t0 = 0; t0 < NB; t0 += 4) {
      double av[4], bv[2];
#pragma unroll
      for (int a = 0; a < 4; a++) av[a] = S0[(t0 + q) * US + wm + 8 * a + g];
#pragma unroll
      for (int b = 0; b < 2; b++) bv[b] = S2[(t0 + q) * US + wn + 8 * b + g];
#pragma unroll
      for (int a = 0; a < 4; a++)
#pragma unroll
        for (int b = 0; b < 2; b++) dmma(acc[a][b][0], acc[a][b][1], av[a], bv[b]);
    }
#pragma unroll
    for (int a = 0; a < 4; a++) {
      const int64_t row = R0 + wm + 8 * a + g;
      if (row < N && row >= rb) {
#pragma unroll
        for (int b = 0; b < 2; b++)
#pragma unroll
          for (int e = 0; e < 2; e++) {
            const int col = wn + 8 * b + 2 * q + e;
            if (col < nbp) {
              f.W[row + col * ldw] = acc[a][b][e];
              f.Lb[row + col * ldw] = acc[a][b][e] * r1s[col];      // speculative L21
              cm[b][e] = fmax(cm[b][e], fabs(acc[a][b][e]));
            }
          }
      }
    }
    __syncthreads();   // S0 is refilled by the next tile
  }
  // per-column max |W21| over this CTA's tiles: reduce over g, then over the two row halves
#pragma unroll
  for (int b = 0; b < 2; b++)
#pragma unroll
    for (int e = 0; e < 2; e++) {
      double v = cm[b][e];
      v = fmax(v, __shfl_xor_sync(0xffffffffu, v, 4));
      v = fmax(v, __shfl_xor_sync(0xffffffffu, v, 8));
      v = fmax(v, __shfl_xor_sync(0xffffffffu, v, 16));
      if (g == 0) cmx[warp][8 * b + 2 * q + e] = v;
    }
  __syncthreads();
  if (tid < NB) {
    const int c = tid, w0 = 2 * (c >> 4);
    const double v = fmax(cmx[w0][c & 15], cmx[w0 + 1][c & 15]);
    if (c < nbp) atomicMax(&ctl->colmax[c], dbits(v));
  }
}

__global__ void __launch_bounds__(256, 1) k_panel_fast(int64_t N, double* __restrict__ A, int64_t lda, FWork f) {
  pdl_wait();
  FCtl* ctl = f.ctl;
  if (ctl->abort) return;
  __shared__ int s_role;
  if (threadIdx.x == 0) s_role = (int)atomicAdd(&f.ucount[3 * f.pidx + 1], 1ull);   // (slot 3q+1: tickets)
  __syncthreads();
  const int role = s_role;
  const int64_t k0 = panel_k0(f);
  if (k0 >= N) {
    if (role == 0 && threadIdx.x == 0) { ctl->k0 = (int)N; ctl->kb = 0; ctl->nbp = 0; }
    return;
  }
  const int nbp = (int)((N - k0) < NB ? (N - k0) : NB);
  const bool fprev = f.fuse && f.pidx > 0;
  extern __shared__ double sm[];
  if (role == 0) f1_body(N, A, lda, f, k0, nbp, fprev, sm);
  else f2_role(N, A, lda, f, k0, nbp, fprev, role, (int)gridDim.x - 1, sm);
}

// F2: W21 = A21 * X (X = L11^{-T}) on the FP64 tensor cores, 64-row tiles,
// K = 64; writes W21, speculative L21 = W21 D^{-1}, and atomically
// max-reduces |W21| per column (colmax).  Tiles are claimed from the panel's
// F2 counter, which the concurrent trailing update (k_update_tma<3, true>) also
// draws from once this panel's X is published: whatever it has not taken is
// done here.
__global__ void __launch_bounds__(128) k_panel_trsm(int64_t N, const double* __restrict__ A, int64_t lda, FWork f) {
  bsel_ws(f, blockIdx.y);
  A += blockIdx.y * f.bms;
  pdl_trigger();   // let k_panel_slow launch and wait (griddepcontrol.wait) behind us
  FCtl* ctl = f.ctl;
  if (ctl->abort) return;
  const int nbp = ctl->nbp;
  const int64_t k0 = ctl->k0;
  if (nbp == 0) return;
  const int64_t rb = k0 + nbp;
  // tiles on the absolute 64-row grid (the same tiling as the F2 tiles of k_update_tma<3, true>,
  // which claims from the same counter); rows < rb are masked
  const int64_t rbase = (rb / UT) * UT;
  const int64_t ntile = (N > rb) ? (N + UT - 1) / UT - rb / UT : 0;
  if ((int64_t)blockIdx.x >= ntile) return;
  unsigned long long* counter = f.ucount + 3 * f.pidx + 2;
  extern __shared__ double dsm[];
  double* As = dsm;                 // [t][row]
  double* Xs = dsm + NB * US;       // [t][j]
  __shared__ double cmax[4][32];
  __shared__ double r1s[NB];
  __shared__ long long s_x;
  const int tid = threadIdx.x;
  if (tid == 0) s_x = (long long)atomicAdd(counter, 1ull);
  __syncthreads();
  long long x = s_x;
  if (tid == 0) UTRACE_MIN(f.pidx, 3);
  if (x >= ntile) { if (tid == 0) UTRACE_MAX(f.pidx, 4); return; }
  if (tid < NB) {
    const double d = (tid < nbp) ? ctl->d[tid] : 0.0;
    r1s[tid] = (d != 0.0) ? fast_rcp(d) : 0.0;
  }
  stage_x<128, false>(Xs, f.Lblk, tid);   // Xs[t * US + i] = X[t][j=i]
  const int warp = tid >> 5, lane = tid & 31;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
  const int g = lane >> 2, q = lane & 3;
  double cm[4][2];
#pragma unroll
  for (int b = 0; b < 4; b++) cm[b][0] = cm[b][1] = 0.0;
  while (x < ntile) {
    const int64_t R0 = rbase + x * UT;
    for (int idx = tid; idx < UT * NB; idx += 128) {
      const int i = idx % UT, t = idx / UT;
      As[t * US + i] = (t < nbp && R0 + i < N && R0 + i >= rb) ? A[(R0 + i) + (k0 + t) * lda] : 0.0;
    }
    __syncthreads();
    if (tid == 0) s_x = (long long)atomicAdd(counter, 1ull);   // next claim (read after the closing barrier)
    double acc[4][4][2];
#pragma unroll
    for (int a = 0; a < 4; a++)
#pragma unroll
      for (int b = 0; b < 4; b++) acc[a][b][0] = acc[a][b][1] = 0.0;
#pragma unroll 4
    for (int t0 = 0; t0 < NB; t0 += 4) {
      double av[4], bv[4];
#pragma unroll
      for (int a = 0; a < 4; a++) av[a] = As[(t0 + q) * US + wm + 8 * a + g];
#pragma unroll
      for (int b = 0; b < 4; b++) bv[b] = Xs[(t0 + q) * US + wn + 8 * b + g];
#pragma unroll
      for (int a = 0; a < 4; a++)
#pragma unroll
        for (int b = 0; b < 4; b++) dmma(acc[a][b][0], acc[a][b][1], av[a], bv[b]);
    }
#pragma unroll
    for (int a = 0; a < 4; a++) {
      const int64_t row = R0 + wm + 8 * a + g;
      if (row < N && row >= rb) {
#pragma unroll
        for (int b = 0; b < 4; b++)
#pragma unroll
          for (int e = 0; e < 2; e++) {
            const int col = wn + 8 * b + 2 * q + e;
            if (col < nbp) {
              f.W[row + col * f.ldw] = acc[a][b][e];
              f.Lb[row + col * f.ldw] = acc[a][b][e] * r1s[col];      // speculative L21
              cm[b][e] = fmax(cm[b][e], fabs(acc[a][b][e]));
            }
          }
      }
    }
    __syncthreads();   // As is refilled; s_x holds the next claim
    if (tid == 0) UTRACE_ADD(f.pidx, 5);
    x = s_x;
  }
  if (tid == 0) UTRACE_MAX(f.pidx, 4);
  // reduce over the 8 row-groups g (lanes with equal q share columns)
#pragma unroll
  for (int b = 0; b < 4; b++)
#pragma unroll
    for (int e = 0; e < 2; e++) {
      double v = cm[b][e];
      v = fmax(v, __shfl_xor_sync(0xffffffffu, v, 4));
      v = fmax(v, __shfl_xor_sync(0xffffffffu, v, 8));
      v = fmax(v, __shfl_xor_sync(0xffffffffu, v, 16));
      if (g == 0) cmax[warp][8 * b + 2 * q + e] = v;
    }
  __syncthreads();
  if (tid < NB) {
    const int col = tid;
    const int half = col >> 5;                 // column col is owned by warps half and half+2
    const double v = fmax(cmax[half][col & 31], cmax[half + 2][col & 31]);
    if (col < nbp) atomicMax(&ctl->colmax[col], dbits(v));
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

// W columns [kb, NB) of rows >= k0 hold speculative / stale values; the TMA
// update multiplies all NB columns, so they must be exactly zero.
__device__ __forceinline__ void zero_w_tail(int64_t N, int64_t k0, int kb, const FWork& f) {
  const int64_t nr = N - k0;
  const int nc = NB - kb;
  if (nr <= 0 || nc <= 0) return;
  for (int64_t idx = threadIdx.x; idx < nr * nc; idx += blockDim.x) {
    const int64_t r = k0 + idx % nr, c = kb + idx / nr;
    f.W[r + c * f.ldw] = 0.0;
    f.Lb[r + c * f.ldw] = 0.0;
  }
}

__global__ void __launch_bounds__(1024) k_panel_slow(int64_t N, double* __restrict__ A, int64_t lda, FWork f,
                                                     int32_t* piv) {
  bsel_ws(f, blockIdx.y);
  A += blockIdx.y * f.bms;
  piv += blockIdx.y * f.bps;
  pdl_wait();
  pdl_trigger();
  FCtl* ctl = f.ctl;
  if (ctl->abort) return;
  const int nbp = ctl->nbp;
  const int64_t k0 = ctl->k0;
  if (nbp == 0) {
    if (threadIdx.x == 0) f.pinfo[f.pidx] = make_int2((int)k0, 0);
    return;
  }
  // accept the longest prefix of columns that pass BK's 1x1-no-interchange test
  // |d_j| >= alpha * colmax_j on the speculatively updated values (all tested in parallel)
  __shared__ unsigned s_fail[2], s_pos[2], s_neg[2];
  double dj = 0.0;
  if (threadIdx.x < NB) {
    const int jj = threadIdx.x;
    dj = (jj < nbp) ? ctl->d[jj] : 0.0;
    const double cm = (jj < nbp) ? bitsd(ctl->colmax[jj]) : 0.0;
    const bool fail = (jj >= nbp) || !(fabs(dj) >= ALPHA_BK * cm);   // (0 >= 0 accepts the exact-zero column)
    const double tol = ctl->tol;
    const unsigned b = __ballot_sync(0xffffffffu, fail);
    const unsigned bp = __ballot_sync(0xffffffffu, dj > tol);
    const unsigned bn = __ballot_sync(0xffffffffu, dj < -tol);
    if ((jj & 31) == 0) { s_fail[jj >> 5] = b; s_pos[jj >> 5] = bp; s_neg[jj >> 5] = bn; }
  }
  __syncthreads();
  const int p = s_fail[0] ? (__ffs(s_fail[0]) - 1) : (s_fail[1] ? 32 + __ffs(s_fail[1]) - 1 : NB);
  if (threadIdx.x < p) piv[k0 + threadIdx.x] = (int32_t)(k0 + threadIdx.x + 1);
  if (threadIdx.x == 0 && p > 0) {
    // inertia of the accepted prefix: popcounts of the sign masks below p
    const unsigned long long m = (p >= 64) ? ~0ull : ((1ull << p) - 1ull);
    const unsigned long long pos = ((unsigned long long)s_pos[1] << 32 | s_pos[0]) & m;
    const unsigned long long neg = ((unsigned long long)s_neg[1] << 32 | s_neg[0]) & m;
    const int np = __popcll(pos), nn = __popcll(neg);
    ctl->inertia[0] += np;
    ctl->inertia[2] += nn;
    ctl->inertia[1] += p - np - nn;
  }
  int j = p;
  const bool last = (k0 + nbp >= N);
  const int jlim = last ? nbp : nbp - 1;
  if (j >= jlim) {   // nothing left for the exact path: publish (k0, kb) for the updates
    if (threadIdx.x == 0) { ctl->kb = j; f.pinfo[f.pidx] = make_int2((int)k0, j); }
    zero_w_tail(N, k0, j, f);
    return;
  }
  __shared__ double wrow[WCOLS];
  __shared__ ArgMax sh[33];
  double* W = f.W;
  double* Lb = f.Lb;
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
      for (int t = 0; t < j; t++) v -= Lb[r + t * ldw] * wrow[t];
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
        for (int t = 0; t < j; t++) v -= Lb[r + t * ldw] * wrow[t];
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
      for (int64_t c = tid; c < kk - k0; c += nth) {
        double t = Lb[kk + c * ldw]; Lb[kk + c * ldw] = Lb[kp + c * ldw]; Lb[kp + c * ldw] = t;
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
      for (int64_t r = k + 1 + tid; r < N; r += nth) Lb[r + j * ldw] = zero ? W[r + j * ldw] : W[r + j * ldw] * r1;
      if (tid == 0) {
        Lb[k + j * ldw] = d;
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
        Lb[r + j * ldw] = d21 * (d11 * wk - wk1);
        Lb[r + (j + 1) * ldw] = d21 * (d22 * wk1 - wk);
      }
      if (tid == 0) {
        Lb[k + j * ldw] = W[k + j * ldw];
        Lb[(k + 1) + j * ldw] = W[(k + 1) + j * ldw];             // D21 (moved to the upper slot at finalize)
        Lb[(k + 1) + (j + 1) * ldw] = W[(k + 1) + (j + 1) * ldw];
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
  if (tid == 0) {
    ctl->kb = j;
    ctl->nexact += j - p;
    f.pinfo[f.pidx] = make_int2((int)k0, j);
  }
  zero_w_tail(N, k0, j, f);
}

// F4, multi-CTA: the same acceptance + exact dlasyf panel as k_panel_slow, but
// the per-column work (two GEMVs against the panel's finished columns, the
// column/row argmax, the interchange and the scaling) is spread over G CTAs
// that each own a contiguous block of rows [k0, N); the BK decisions need the
// global column max, so CTAs meet at a grid barrier after each argmax (every
// CTA then takes the same decision from the same partials, in fixed order) and
// once more after an interchange.  One CTA did one column in ~55 us at
// N = 32768 (the GEMVs stream ~4-8 MB of L2 each); this takes a few us.
// All CTAs must be co-resident: G <= the SM count, launched only after the
// trailing update it depends on has finished (its successors are launched
// programmatically after every CTA here has started).  Cross-CTA data is read
// with ld.global.cg (L2), never through L1.
// Grid barrier + argmax exchange: every CTA stores its partial (v, i) in its
// slot of the bank of this barrier's parity, then arrives on the panel's
// counter (release) and thread 0 spins until all G CTAs have arrived
// (acquire); the G partials are then reduced in fixed order by every CTA.
// (A variant where every CTA polled all G tagged records was slower: 128x
// more pollers on L2.)  Banks alternate by barrier parity, so a CTA that runs
// ahead never overwrites a partial another CTA has yet to read.
// pay / pay_owner / pay_out: the two payload doubles CTA pay_owner wrote into its slot of
// this exchange's payload bank (before the exchange) are read with the partials (same
// round trip) and left in pay_out (shared memory) for every thread.
__device__ __forceinline__ ArgMax x_exchange(unsigned* ctr, ArgMax* part, unsigned& nbar, ArgMax mine, ArgMax* sh,
                                             const double* pay = nullptr, int pay_owner = -1,
                                             double* pay_out = nullptr) {
  const unsigned bk = nbar & 1u;
  ArgMax* bank = part + XMAXG * bk;
  if (threadIdx.x == 0) bank[blockIdx.x] = mine;
  __syncthreads();   // every global write of this CTA precedes the release below
  nbar++;
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;\n" ::"l"(ctr) : "memory");
    const unsigned target = nbar * gridDim.x;
    while (ld_acquire_u32(ctr) < target) {
    }
  }
  __syncthreads();
  ArgMax a{-1.0, 0x7fffffff};
  for (int c = threadIdx.x; c < (int)gridDim.x; c += blockDim.x) {
    a = am_better(a, ArgMax{__ldcg(&bank[c].v), __ldcg(&bank[c].i)});
    if (c == pay_owner) {
      const double* ps = pay + ((size_t)bk * XMAXG + c) * 2;
      pay_out[0] = __ldcg(ps);
      pay_out[1] = __ldcg(ps + 1);
    }
  }
  return block_argmax(a, sh);   // (its block barriers publish pay_out)
}

// The same exchange inside ONE thread-block cluster (the exact panel launched as a
// cluster of G <= 16 CTAs): the argmax partials go to CTA 0's shared memory over DSMEM
// and the hardware cluster barrier (release / acquire at cluster scope, global memory
// included) replaces the global counter -- ~0.7 instead of ~1.75 us (tools/barrier_bench).
// The payloads stay in global memory (ordered by the same barrier).
constexpr int XCL = 16;
struct ClBank {
  ArgMax rec[2][XCL];
};
__device__ __forceinline__ ArgMax x_exchange_cl(ClBank* local, unsigned& nbar, ArgMax mine, ArgMax* sh,
                                                const double* pay = nullptr, int pay_owner = -1,
                                                double* pay_out = nullptr) {
  cg::cluster_group cl = cg::this_cluster();
  const unsigned bk = nbar & 1u;
  ClBank* b0 = cl.map_shared_rank(local, 0);
  if (threadIdx.x == 0) b0->rec[bk][cl.block_rank()] = mine;
  nbar++;
  cl.sync();
  ArgMax a{-1.0, 0x7fffffff};
  const int G = (int)cl.num_blocks();
  for (int c = threadIdx.x; c < G; c += blockDim.x) {
    a = am_better(a, b0->rec[bk][c]);
    if (c == pay_owner) {
      const double* ps = pay + ((size_t)bk * XMAXG + c) * 2;
      pay_out[0] = __ldcg(ps);
      pay_out[1] = __ldcg(ps + 1);
    }
  }
  return block_argmax(a, sh);
}

// own rows r in [rlo, rhi), r >= k:  W(r, wcol) = a_r - sum_{t<j} Lb(r, t) wv[t], with
// a_r = A(r, kc) (column kc; for IMAX the row/column kc = imax of the lower triangle);
// a quad of threads per row (t strided by 4, fixed-order shuffle sum).  Returns the CTA's
// argmax of |W(r, wcol)| over r > k (column) or r != kc (IMAX).
template <bool IMAX>
__device__ __forceinline__ ArgMax x_gemv(const double* A, int64_t lda, const double* Lb, double* W, int64_t ldw,
                                         int64_t rlo, int64_t rhi, int64_t k, int64_t kc, int j, int wcol,
                                         const double* wv, double* aux, const double* Ls, int lstr) {
  const int tid = threadIdx.x, qd = tid & 3;
  ArgMax am{-1.0, 0x7fffffff};
  const int64_t rfirst = rlo + ((k > rlo) ? ((k - rlo) / XROWS) * XROWS : 0);
  for (int64_t rb = rfirst; rb < rhi; rb += XROWS) {
    const int64_t r = rb + (tid >> 2);
    const bool live = r < rhi && r >= k;
    double a = 0.0;   // issued before the dot product (its latency overlaps it)
    if (live && qd == 0)
      a = IMAX ? ((r < kc) ? __ldcg(&A[kc + r * lda]) : __ldcg(&A[r + kc * lda])) : __ldcg(&A[r + kc * lda]);
    double s0 = 0.0, s1 = 0.0;
    if (live && Ls) {   // the CTA's rows of the panel's finished columns, kept in shared memory
      const double* lr = Ls + (r - rlo);
      int t = qd;
      for (; t + 4 < j; t += 8) {
        s0 = fma(lr[t * lstr], wv[t], s0);
        s1 = fma(lr[(t + 4) * lstr], wv[t + 4], s1);
      }
      if (t < j) s0 = fma(lr[t * lstr], wv[t], s0);
    } else if (live) {
      const double* lr = Lb + r;
      int t = qd;
      for (; t + 4 < j; t += 8) {
        s0 = fma(__ldcg(lr + (int64_t)t * ldw), wv[t], s0);
        s1 = fma(__ldcg(lr + (int64_t)(t + 4) * ldw), wv[t + 4], s1);
      }
      if (t < j) s0 = fma(__ldcg(lr + (int64_t)t * ldw), wv[t], s0);
    }
    double s = s0 + s1;
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    if (live && qd == 0) {
      const double v = a - s;
      W[r + wcol * ldw] = v;
      if (IMAX ? (r != kc) : (r > k)) am = am_better(am, ArgMax{fabs(v), (int)r});
      // payload of the row the decision needs, published through the exchange (no reload):
      // W(k, j) by the owner of row k; W(imax, j+1) and W(imax, j) by the owner of row imax
      if (!IMAX && r == k) aux[0] = v;
      if (IMAX && r == kc) { aux[0] = v; aux[1] = __ldcg(&W[r + (wcol - 1) * ldw]); }
    }
  }
  return am;
}

// F2 tiles the concurrent trailing update did not take (it claims them only once X
// is published and never waits for it): W21 = A21 X, L21 = W21 D^{-1}, colmax -- the
// same arithmetic as k_panel_trsm, on warps 0-3 of a k_panel_exact CTA.  Tiles
// [c0, ntile) are dealt to the CTAs statically (the claim counter is stable: the
// update that claims from it has finished before this kernel starts).
__device__ __noinline__ void x_f2_leftovers(int64_t N, const double* __restrict__ A, int64_t lda, const FWork& f,
                                            int64_t k0, int nbp, int64_t c0, int64_t ntile, double* sm) {
  FCtl* ctl = f.ctl;
  const int64_t rb = k0 + nbp;
  const int64_t rbase = (rb / UT) * UT;
  double* As = sm;                 // [t][row]
  double* Xs = sm + NB * US;       // [t][j]
  __shared__ double cmax[4][32];
  __shared__ double r1s[NB];
  const int tid = threadIdx.x;
  if (tid < NB) {
    const double d = (tid < nbp) ? __ldcg(&ctl->d[tid]) : 0.0;
    r1s[tid] = (d != 0.0) ? fast_rcp(d) : 0.0;
  }
  stage_x<XT, true>(Xs, f.Lblk, tid);
  const int warp = tid >> 5, lane = tid & 31;
  const int wm = ((warp & 3) >> 1) * 32, wn = (warp & 1) * 32;
  const int g = lane >> 2, q = lane & 3;
  double cm[4][2];
#pragma unroll
  for (int b = 0; b < 4; b++) cm[b][0] = cm[b][1] = 0.0;
  for (int64_t x = c0 + blockIdx.x; x < ntile; x += gridDim.x) {
    const int64_t R0 = rbase + x * UT;
    __syncthreads();   // (Xs / r1s ready; As free)
    for (int idx = tid; idx < UT * NB; idx += XT) {
      const int i = idx % UT, t = idx / UT;
      As[t * US + i] = (t < nbp && R0 + i < N && R0 + i >= rb) ? __ldcg(&A[(R0 + i) + (k0 + t) * lda]) : 0.0;
    }
    __syncthreads();
    if (warp < 4) {
      double acc[4][4][2];
#pragma unroll
      for (int a = 0; a < 4; a++)
#pragma unroll
        for (int b = 0; b < 4; b++) acc[a][b][0] = acc[a][b][1] = 0.0;
#pragma unroll 4
      for (int t0 = 0; t0 < NB; t0 += 4) {
        double av[4], bv[4];
#pragma unroll
        for (int a = 0; a < 4; a++) av[a] = As[(t0 + q) * US + wm + 8 * a + g];
#pragma unroll
        for (int b = 0; b < 4; b++) bv[b] = Xs[(t0 + q) * US + wn + 8 * b + g];
#pragma unroll
        for (int a = 0; a < 4; a++)
#pragma unroll
          for (int b = 0; b < 4; b++) dmma(acc[a][b][0], acc[a][b][1], av[a], bv[b]);
      }
#pragma unroll
      for (int a = 0; a < 4; a++) {
        const int64_t row = R0 + wm + 8 * a + g;
        if (row < N && row >= rb) {
#pragma unroll
          for (int b = 0; b < 4; b++)
#pragma unroll
            for (int e = 0; e < 2; e++) {
              const int col = wn + 8 * b + 2 * q + e;
              if (col < nbp) {
                f.W[row + col * f.ldw] = acc[a][b][e];
                f.Lb[row + col * f.ldw] = acc[a][b][e] * r1s[col];
                cm[b][e] = fmax(cm[b][e], fabs(acc[a][b][e]));
              }
            }
        }
      }
    }
  }
  if (warp < 4) {
#pragma unroll
    for (int b = 0; b < 4; b++)
#pragma unroll
      for (int e = 0; e < 2; e++) {
        double v = cm[b][e];
        v = fmax(v, __shfl_xor_sync(0xffffffffu, v, 4));
        v = fmax(v, __shfl_xor_sync(0xffffffffu, v, 8));
        v = fmax(v, __shfl_xor_sync(0xffffffffu, v, 16));
        if (g == 0) cmax[warp][8 * b + 2 * q + e] = v;
      }
  }
  __syncthreads();
  if (tid < NB && c0 + blockIdx.x < ntile) {
    const int col = tid, half = col >> 5;
    const double v = fmax(cmax[half][col & 31], cmax[half + 2][col & 31]);
    if (col < nbp) atomicMax(&ctl->colmax[col], dbits(v));
  }
}

template <bool CL>
__global__ void __launch_bounds__(XT) k_panel_exact(int64_t N, double* __restrict__ A, int64_t lda, FWork f,
                                                    int32_t* piv, int xchunk, int use_ls, int f2left) {
  bsel_ws(f, blockIdx.y);
  A += blockIdx.y * f.bms;
  piv += blockIdx.y * f.bps;
  pdl_wait();
  pdl_trigger();
  F4TRACE_MIN(f.pidx);
  FCtl* ctl = f.ctl;
  if (ctl->abort) return;
  const int nbp = ctl->nbp;
  const int64_t k0 = ctl->k0;
  const int tid = threadIdx.x;
  const bool c0 = (blockIdx.x == 0);
  if (nbp == 0) {
    if (c0 && tid == 0) f.pinfo[f.pidx] = make_int2((int)k0, 0);
    return;
  }
  extern __shared__ double xls[];
  __shared__ ArgMax sh[33];
  __shared__ double s_pay[2];
  __shared__ ClBank clb;             // (CL: CTA 0's copy receives the partials)
  unsigned* ctr = f.xbar + f.pidx;   // this panel's barrier counter (zeroed by k_factor_init)
  unsigned nbar = 0;                 // barriers so far
  // grid exchange: the global counter, or the cluster barrier (CL)
  auto xch = [&](ArgMax mine, const double* pay, int owner, double* out) -> ArgMax {
    if constexpr (CL) return x_exchange_cl(&clb, nbar, mine, sh, pay, owner, out);
    else return x_exchange(ctr, f.xpart, nbar, mine, sh, pay, owner, out);
  };
  if (f2left) {
    // this panel's F2 tiles the previous panel's trailing update did not take (replaces a
    // separate k_panel_trsm launch on the critical hand-off); colmax is complete after the barrier
    const int64_t rb = k0 + nbp;
    const int64_t ntile = (N > rb) ? (N + UT - 1) / UT - rb / UT : 0;
    const unsigned long long claimed = __ldcg(f.ucount + 3 * f.pidx + 2);
    const int64_t cfirst = (claimed < (unsigned long long)ntile) ? (int64_t)claimed : ntile;
    if (cfirst < ntile) {
      x_f2_leftovers(N, A, lda, f, k0, nbp, cfirst, ntile, xls);
      xch(ArgMax{-1.0, 0x7fffffff}, nullptr, -1, nullptr);
    }
  }
  // ---- accepted prefix (every CTA computes p; CTA 0 records it)
  __shared__ unsigned s_fail[2], s_pos[2], s_neg[2];
  if (tid < NB) {
    const int jj = tid;
    const double dj = (jj < nbp) ? ctl->d[jj] : 0.0;
    const double cm = (jj < nbp) ? bitsd(__ldcg(&ctl->colmax[jj])) : 0.0;
    const bool fail = (jj >= nbp) || !(fabs(dj) >= ALPHA_BK * cm);
    const double tol = ctl->tol;
    const unsigned b = __ballot_sync(0xffffffffu, fail);
    const unsigned bp = __ballot_sync(0xffffffffu, dj > tol);
    const unsigned bn = __ballot_sync(0xffffffffu, dj < -tol);
    if ((jj & 31) == 0) { s_fail[jj >> 5] = b; s_pos[jj >> 5] = bp; s_neg[jj >> 5] = bn; }
  }
  __syncthreads();
  const int p = s_fail[0] ? (__ffs(s_fail[0]) - 1) : (s_fail[1] ? 32 + __ffs(s_fail[1]) - 1 : NB);
  if (c0) {
    if (tid < p) piv[k0 + tid] = (int32_t)(k0 + tid + 1);
    if (tid == 0 && p > 0) {
      const unsigned long long m = (p >= 64) ? ~0ull : ((1ull << p) - 1ull);
      const unsigned long long pos = ((unsigned long long)s_pos[1] << 32 | s_pos[0]) & m;
      const unsigned long long neg = ((unsigned long long)s_neg[1] << 32 | s_neg[0]) & m;
      const int np = __popcll(pos), nn = __popcll(neg);
      ctl->inertia[0] += np;
      ctl->inertia[2] += nn;
      ctl->inertia[1] += p - np - nn;
    }
  }
  int j = p;
  const bool last = (k0 + nbp >= N);
  const int jlim = last ? nbp : nbp - 1;
  double* W = f.W;
  double* Lb = f.Lb;
  const int64_t ldw = f.ldw;
  if (j < jlim) {
    __shared__ double wrow[WCOLS];
    const double tol = ctl->tol;
    const int64_t chunk = xchunk;   // host: >= ceil((N - k0) / G), multiple of 32
    // the CTA's rows of L (panel columns) in shared memory: Ls[t * lstr + row - rlo]
    // (lstr = 8 mod 16: the 4 k-lanes of a quad fall in opposite bank halves pairwise)
    const int lstr = xchunk + 8;
    const double* Ls = use_ls ? xls : nullptr;
    const int64_t rlo = k0 + (int64_t)blockIdx.x * chunk;
    const int64_t rhi = (rlo + chunk < N) ? rlo + chunk : N;
    if (use_ls) {
      const int64_t nr = rhi - rlo;
      for (int64_t idx = tid; idx < nr * j; idx += XT) {
        const int64_t rl = idx % nr, t = idx / nr;
        xls[t * lstr + rl] = __ldcg(&Lb[(rlo + rl) + t * ldw]);
      }
      __syncthreads();
    }
    while (j < jlim) {
      XPH_DECL;
      const int64_t k = k0 + j;
      for (int t = tid; t < j; t += XT) wrow[t] = __ldcg(&W[k + t * ldw]);
      __syncthreads();
      XPH(0);
      // W(k:N, j) = A(k:N, k) - L(k:N, panel) W(k, panel)^T ; colmax / imax below k
      double* myslot = f.xpay + ((size_t)(nbar & 1u) * XMAXG + blockIdx.x) * 2;
      ArgMax am = x_gemv<false>(A, lda, Lb, W, ldw, rlo, rhi, k, k, j, j, wrow, myslot, Ls, lstr);
      XPH(1);
      am = block_argmax(am, sh);
      XPH(2);
      am = xch(am, f.xpay, (int)((k - k0) / chunk), s_pay);
      XPH(3);
      const double wkk = s_pay[0];   // W(k, j), from the owner of row k
      const double absakk = fabs(wkk);
      double wij1 = 0.0, wij = 0.0;   // W(imax, j+1), W(imax, j) (candidate path)
      const double colmax = (am.v < 0.0) ? 0.0 : am.v;
      const int64_t imax = (am.v < 0.0) ? k : am.i;
      int kstep = 1;
      int64_t kp = k;
      bool zero = false, cand = false;   // cand: the pivot column is W(:, j+1) (1x1 with kp = imax)
      if (fmax(absakk, colmax) == 0.0) {
        zero = true;
      } else if (absakk >= ALPHA_BK * colmax) {
        kp = k;
      } else {
        for (int t = tid; t < j; t += XT) wrow[t] = __ldcg(&W[imax + t * ldw]);
        __syncthreads();
        // candidate column imax, updated: W(k:N, j+1); W(imax, j+1) and W(imax, j) published by its owner
        double* pslot = f.xpay + ((size_t)(nbar & 1u) * XMAXG + blockIdx.x) * 2;
        ArgMax rm = x_gemv<true>(A, lda, Lb, W, ldw, rlo, rhi, k, imax, j, j + 1, wrow, pslot, Ls, lstr);
        rm = block_argmax(rm, sh);
        rm = xch(rm, f.xpay, (int)((imax - k0) / chunk), s_pay);
        const double rowmax = (rm.v < 0.0) ? 0.0 : rm.v;
        wij1 = s_pay[0];
        wij = s_pay[1];
        const double wii = fabs(wij1);
        if (absakk >= ALPHA_BK * colmax * (colmax / rowmax)) {
          kp = k;
        } else if (wii >= ALPHA_BK * rowmax) {
          kp = imax;
          cand = true;
        } else {
          kp = imax;
          kstep = 2;
        }
      }
      XPH(4);   // (the candidate path, when taken)
      const int64_t kk = k + kstep - 1;
      if (kp != kk) {
        // symmetric interchange kk <-> kp of the not-yet-factored part: owners of rows r
        for (int64_t r = rlo + tid; r < rhi; r += XT) {
          if (r <= kk) continue;
          if (r < kp) A[kp + r * lda] = __ldcg(&A[r + kk * lda]);
          else if (r > kp) A[r + kp * lda] = __ldcg(&A[r + kk * lda]);
          // 1x1 with kp = imax: the pivot column is the candidate column (rows kk, kp: below)
          if (cand && r != kp) W[r + j * ldw] = __ldcg(&W[r + (j + 1) * ldw]);
        }
        if (c0) {
          if (tid == 0) { A[kp + kp * lda] = __ldcg(&A[kk + kk * lda]); f.sw[kk] = (int)kp; ctl->nswap += 1; }
          // rows kk <-> kp of the panel's finished L columns and of W (column j from the candidate if cand)
          const int nl = (int)(kk - k0), nw = (int)(kk - k0) + 1;
          for (int c = tid; c < nl + nw; c += XT) {
            if (c < nl) {
              const double a = __ldcg(&Lb[kk + c * ldw]), b = __ldcg(&Lb[kp + c * ldw]);
              Lb[kk + c * ldw] = b;
              Lb[kp + c * ldw] = a;
            } else {
              const int t = c - nl;
              const int ts = (cand && t == j) ? j + 1 : t;
              const double a = __ldcg(&W[kk + ts * ldw]), b = __ldcg(&W[kp + ts * ldw]);
              W[kk + t * ldw] = b;
              W[kp + t * ldw] = a;
            }
          }
        }
        xch(ArgMax{-1.0, 0x7fffffff}, nullptr, -1, nullptr);
        if (use_ls) {   // rows kk / kp of L were swapped by CTA 0: refresh this CTA's copies
          const int nl = j;   // finished columns (column j itself is rewritten by the scaling below)
          for (int c = tid; c < 2 * nl; c += XT) {
            const int64_t r = (c < nl) ? kk : kp;
            const int t = (c < nl) ? c : c - nl;
            if (r >= rlo && r < rhi) xls[t * lstr + (r - rlo)] = __ldcg(&Lb[r + t * ldw]);
          }
          // (ordered before the next GEMV by the barriers below)
        }
      }
      XPH(5);   // (the interchange, when taken)
      if (kstep == 1) {
        const double d = cand ? wij1 : wkk;   // W(k, j) after the interchange (the candidate column's W(imax, j+1) if cand)
        const double r1 = zero ? 0.0 : 1.0 / d;
        for (int64_t r = rlo + tid; r < rhi; r += XT) {
          if (r <= k) continue;
          const double w = __ldcg(&W[r + j * ldw]);
          const double l = zero ? w : w * r1;
          Lb[r + j * ldw] = l;
          if (use_ls) xls[j * lstr + (r - rlo)] = l;
        }
        if (c0 && tid == 0) {
          Lb[k + j * ldw] = d;
          if (d > tol) ctl->inertia[0]++;
          else if (d < -tol) ctl->inertia[2]++;
          else ctl->inertia[1]++;
          piv[k] = (int32_t)(kp + 1);
          f.bt[k] = 0;
        }
      } else {
        // rows k+1 <-> kp = imax interchanged: W(k+1, j) = W(imax, j), W(k+1, j+1) = W(imax, j+1)
        const double w21 = wij;
        const double w22 = wij1;
        const double w11 = wkk;
        double d21 = w21;
        const double d11 = w22 / d21;
        const double d22 = w11 / d21;
        const double tt = 1.0 / (d11 * d22 - 1.0);
        d21 = tt / d21;
        for (int64_t r = rlo + tid; r < rhi; r += XT) {
          if (r < k + 2) continue;
          const double wk = __ldcg(&W[r + j * ldw]), wk1 = __ldcg(&W[r + (j + 1) * ldw]);
          const double l0 = d21 * (d11 * wk - wk1), l1 = d21 * (d22 * wk1 - wk);
          Lb[r + j * ldw] = l0;
          Lb[r + (j + 1) * ldw] = l1;
          if (use_ls) { xls[j * lstr + (r - rlo)] = l0; xls[(j + 1) * lstr + (r - rlo)] = l1; }
        }
        if (c0 && tid == 0) {
          Lb[k + j * ldw] = w11;
          Lb[(k + 1) + j * ldw] = w21;             // D21 (moved to the upper slot at finalize)
          Lb[(k + 1) + (j + 1) * ldw] = w22;
          ctl->inertia[0]++;
          ctl->inertia[2]++;
          piv[k] = piv[k + 1] = (int32_t)(-(kp + 1));
          f.bt[k] = 1;
          f.bt[k + 1] = 2;
        }
      }
      XPH(6);   // scaling
      __syncthreads();
      XPH(7);
      if (threadIdx.x == 0 && blockIdx.x == 0) XPH_COUNT;
      j += kstep;
    }
  }
  if (c0 && tid == 0) {
    ctl->kb = j;
    ctl->nexact += j - p;
    f.pinfo[f.pidx] = make_int2((int)k0, j);
  }
  // W / Lb columns [j, NB) of rows >= k0 must be exactly zero for the TMA update (grid-strided)
  const int64_t nr = N - k0;
  const int nc = NB - j;
  if (nr > 0 && nc > 0) {
    const int64_t gt = (int64_t)blockIdx.x * XT + tid, gs = (int64_t)gridDim.x * XT;
    for (int64_t idx = gt; idx < nr * nc; idx += gs) {
      const int64_t r = k0 + idx % nr, c = j + idx / nr;
      f.W[r + c * ldw] = 0.0;
      f.Lb[r + c * ldw] = 0.0;
    }
  }
  if constexpr (CL) cg::this_cluster().sync();   // CTA 0's shared bank outlives every reader
  F4TRACE_MAX(f.pidx);
}

// Copy the finished panel (D + L columns, rows >= the diagonal) from Lb into M.
__global__ void __launch_bounds__(256) k_panel_store(int64_t N, double* __restrict__ A, int64_t lda, FWork f) {
  bsel_ws(f, blockIdx.z);
  A += blockIdx.z * f.bms;
  if (f.ctl->abort) return;
  const int2 pi = f.pinfo[f.pidx];
  const int64_t k0 = pi.x;
  const int kb = pi.y;
  const int64_t r = k0 + (int64_t)blockIdx.x * 256 + threadIdx.x;
  if (kb <= 0 || r >= N) return;
  const int t0 = blockIdx.y * (NB / 8), t1 = min(kb, t0 + NB / 8);
  for (int t = t0; t < t1; t++)
    if (r >= k0 + t) A[r + (k0 + t) * lda] = f.Lb[r + t * f.ldw];
}

// ---------------------------------------------------------------------------
// Trailing update C -= L21 * W21^T on the lower triangle, FP64 tensor cores.
// Persistent: one 128-thread CTA per SM walks the lower-triangular 64x64 tile
// list (linear order, so concurrently active tiles share their L21 row panel
// in L2).  Each tile's operands -- the L tile (64 x kb), the W tile (64 x kb)
// and the C tile (64 x 64) -- are staged in shared memory with cp.async into a
// 2-stage ring, so the loads of tile t+1 fly while tile t runs on the DMMA
// pipe (mma.sync.m8n8k4.f64 -> SASS DMMA.8x8x4; 4 warps of 32x32, K = kb <= 64
// in one pass, C accumulated in registers, stored straight back to HBM).
constexpr int UCS = UT + 2;                         // C tile stride (conflict-free fragment reads)
constexpr int USTAGE = 2 * NB * US + UT * UCS;      // doubles per stage

__device__ __forceinline__ void cp_async8(double* sdst, const double* gsrc, bool pred) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
  const int sz = pred ? 8 : 0;   // src-size 0 -> zero fill
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gsrc), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_async16(double* sdst, const double* gsrc, int bytes) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gsrc), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int NPEND>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(NPEND) : "memory"); }

__device__ __forceinline__ void tri_tile(int64_t x, int64_t& bi, int64_t& bj) {
  bi = (int64_t)((sqrt(8.0 * (double)x + 1.0) - 1.0) * 0.5);
  while (bi * (bi + 1) / 2 > x) bi--;
  while ((bi + 1) * (bi + 2) / 2 <= x) bi++;
  bj = x - bi * (bi + 1) / 2;
}

// Tiles are anchored on the ABSOLUTE 64-grid (tile (BI,BJ) covers rows
// [64 BI, 64 BI + 64) x cols [64 BJ, 64 BJ + 64)), so with a 16-byte aligned
// M and even ldm every tile column segment is 16-byte aligned: one 16-byte
// cp.async moves two doubles.  Rows/cols < s (already factored) are computed
// on but never stored.
template <bool V16>
__device__ __forceinline__ void update_issue(double* st, int64_t R0, int64_t C0, int64_t k0, int kb, int kp4,
                                             int64_t N, const double* A, int64_t lda, const double* W,
                                             int64_t ldw, const double* Lp) {
  double* Ls = st;
  double* Ws = st + NB * US;
  double* Cs = st + 2 * NB * US;
  if (V16) {
    // pairs of rows: idx -> (pair ip = idx & 31, column t = idx >> 5)
    const int ip = threadIdx.x & 31;
    const int i = 2 * ip;
    const int64_t ra = R0 + i, ca = C0 + i;
    const int64_t dl = N - ra, dw = N - ca;
    const int nl = (dl >= 2) ? 16 : (dl == 1 ? 8 : 0);
    const int nw = (dw >= 2) ? 16 : (dw == 1 ? 8 : 0);
    const double* gl = Lp + ra;
    const double* gw = W + ca;
    for (int t = threadIdx.x >> 5; t < kp4; t += 4) {
      const bool tin = t < kb;
      cp_async16(&Ls[t * US + i], (tin && nl) ? gl + t * ldw : Lp, tin ? nl : 0);
      cp_async16(&Ws[t * US + i], (tin && nw) ? gw + t * ldw : W, tin ? nw : 0);
    }
    const double* gc = A + ra + C0 * lda;
    for (int c = threadIdx.x >> 5; c < UT; c += 4) {
      const int nc = (C0 + c < N) ? nl : 0;
      cp_async16(&Cs[c * UCS + i], nc ? gc + c * lda : A, nc);
    }
  } else {
    for (int idx = threadIdx.x; idx < UT * kp4; idx += 128) {
      const int i = idx & (UT - 1), t = idx >> 6;
      const bool tin = t < kb;
      const bool pl = tin && (R0 + i < N), pw = tin && (C0 + i < N);
      cp_async8(&Ls[t * US + i], pl ? &Lp[(R0 + i) + t * ldw] : Lp, pl);
      cp_async8(&Ws[t * US + i], pw ? &W[(C0 + i) + t * ldw] : W, pw);
    }
    for (int idx = threadIdx.x; idx < UT * UT; idx += 128) {
      const int i = idx & (UT - 1), c = idx >> 6;
      const bool pc = (R0 + i < N) && (C0 + c < N);
      cp_async8(&Cs[c * UCS + i], pc ? &A[(R0 + i) + (C0 + c) * lda] : A, pc);
    }
  }
}

template <bool V16>
__global__ void __launch_bounds__(128, 1) k_update(int64_t N, double* __restrict__ A, int64_t lda, FWork f) {
  FCtl* ctl = f.ctl;
  if (ctl->abort) return;
  const int2 pi = f.pinfo[f.pidx];
  const int64_t k0 = pi.x;
  const int kb = pi.y;
  const int64_t s = k0 + kb;
  if (N - s <= 0 || kb <= 0) return;
  const int64_t b0 = s / UT;                               // first absolute tile row/col
  const int64_t nt = (N + UT - 1) / UT - b0;
  const int64_t ntiles = nt * (nt + 1) / 2;
  int64_t x = blockIdx.x;
  if (x >= ntiles) return;
  extern __shared__ double sm[];
  const int kp4 = (kb + 3) & ~3;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
  const int g = lane >> 2, q = lane & 3;
  int64_t bi, bj;
  tri_tile(x, bi, bj);
  int64_t R0 = (b0 + bi) * UT, C0 = (b0 + bj) * UT;
  update_issue<V16>(sm, R0, C0, k0, kb, kp4, N, A, lda, f.W, f.ldw, f.Lb);
  cp_async_commit();
  for (int it = 0; x < ntiles; it++) {
    const int64_t xn = x + gridDim.x;
    double* cur = sm + (size_t)(it & 1) * USTAGE;
    int64_t Rn = 0, Cn = 0;
    if (xn < ntiles) {
      int64_t bin, bjn;
      tri_tile(xn, bin, bjn);
      Rn = (b0 + bin) * UT; Cn = (b0 + bjn) * UT;
      update_issue<V16>(sm + (size_t)((it + 1) & 1) * USTAGE, Rn, Cn, k0, kb, kp4, N, A, lda, f.W, f.ldw, f.Lb);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double* Ls = cur;
    const double* Ws = cur + NB * US;
    const double* Cs = cur + 2 * NB * US;
    double acc[4][4][2];
#pragma unroll
    for (int a = 0; a < 4; a++)
#pragma unroll
      for (int b = 0; b < 4; b++)
#pragma unroll
        for (int e = 0; e < 2; e++) acc[a][b][e] = Cs[(wn + 8 * b + 2 * q + e) * UCS + wm + 8 * a + g];
#pragma unroll 4
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
    for (int a = 0; a < 4; a++) {
      const int64_t row = R0 + wm + 8 * a + g;
#pragma unroll
      for (int b = 0; b < 4; b++)
#pragma unroll
        for (int e = 0; e < 2; e++) {
          const int64_t col = C0 + wn + 8 * b + 2 * q + e;
          if (row < N && col >= s && row >= col) A[row + col * lda] = acc[a][b][e];
        }
    }
    __syncthreads();   // stage `cur` may be refilled by the next iteration's issue
    x = xn; R0 = Rn; C0 = Cn;
  }
}

// ---------------------------------------------------------------------------
// Trailing update, TMA + warp-specialised version (the default when M is
// 16-byte aligned with an even ldm).  One producer warp issues
// cp.async.bulk.tensor (TMA, SASS UTMALDG) copies of the L21 and W21 tiles
// into a 3-stage shared-memory ring (64-byte swizzle: conflict-free DMMA
// fragment reads), completion tracked by mbarriers; two consumer groups of
// 4 warps each take alternate tiles ("ping-pong"), so one group's C loads
// and epilogue stores overlap the other group's DMMA k-loop.
constexpr int TNG = 2;                            // consumer groups (4 warps each), ping-pong
constexpr int TSMAX = 3;                          // pipeline stages (L + W tiles) -- in-place staging variant
constexpr int TTHREADS = 32 * (1 + 4 * TNG);      // producer warp + consumer warps
constexpr int TOPB = UT * NB * 8;                 // bytes per operand tile (32 KB)
constexpr int TSTAGEB = 2 * TOPB;                 // L + W
constexpr int TBOXB = 16 * NB * 8;                // bytes per TMA box (16 rows x 64 k, 8 KB)
// OUTB variant: 2 stages + one 32 KB output buffer per consumer group (a stage is released as soon as
// its k-loop is done); in-place variant: 3 stages, -P staged in the consumed stage (released after the
// TMA reduce has read it).  Both use 192 KB.
constexpr int TSMEM = TSMAX * TSTAGEB + 1024 + 16 * TSMAX + 16 * TSMAX;   // + alignment + barriers + 2 tile slots

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(bar), "r"(parity) : "memory");
}
__device__ __forceinline__ void tma_load_2d(unsigned dst, const CUtensorMap* map, int c0, int c1, unsigned bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(dst),
      "l"(map), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
// byte offset of element (row i in 0..63, k t in 0..63) inside an operand tile:
// 4 boxes of 16 rows x 64 k (8 KB each), 128-byte swizzle (bits[4:6] ^= bits[7:9]).
// (16-row boxes: the TMA engine moves 128-byte rows, 1.45x the load throughput
// of 8-row / 64-byte boxes -- tools/tma_bw_probe.cu: 50 vs 35 B/clk/SM -- and the
// operand loads share it with the reduce-add of the result tile.)
__device__ __forceinline__ unsigned tma_off(int i, int t) {
  const unsigned lin = (unsigned)(t * 128 + (i & 15) * 8);
  return (unsigned)((i >> 4) * TBOXB) + (lin ^ (((lin >> 7) & 7u) << 4));
}

// Tile sets: mode 0 = all lower tiles of the trailing matrix (columns >= s).
// Look-ahead (mode 3; nbn = width of the next panel, which starts at column
// s): the same set minus the next panel's diagonal block (k_panel_diag
// updates that itself), in the order: tile column b0, tile column b0+1 (the
// "T1" tiles, which hold the next panel's columns), then the rest -- so the
// dynamic queue finishes the next panel's columns first.
// mode 4 (tail panels, whose F2 tiles apply the deferred update themselves):
// tile column b0+1, then the rest; columns >= s+nbn only.
__device__ __forceinline__ int64_t upd_nt1(int64_t nt, int mode) {
  if (mode == 4) return nt >= 2 ? nt - 1 : 0;
  return nt >= 2 ? 2 * nt - 1 : nt;
}
__device__ __forceinline__ int64_t upd_ntiles(int64_t nt, int mode) {
  if (mode == 0) return nt * (nt + 1) / 2;
  const int64_t r = nt - 2;
  return upd_nt1(nt, mode) + (r > 0 ? r * (r + 1) / 2 : 0);
}
__device__ __forceinline__ void upd_tile(int64_t x, int64_t nt, int mode, int64_t& bi, int64_t& bj) {
  if (mode == 0) { tri_tile(x, bi, bj); return; }
  if (mode == 3) {
    if (x < nt) { bi = x; bj = 0; return; }
    if (x < upd_nt1(nt, 3)) { bi = x - nt + 1; bj = 1; return; }
  } else {
    if (x < upd_nt1(nt, 4)) { bi = x + 1; bj = 1; return; }
  }
  tri_tile(x - upd_nt1(nt, mode), bi, bj);
  bi += 2; bj += 2;
}
// entries (row, col) a launch of this mode may change
__device__ __forceinline__ bool upd_mask(int64_t row, int64_t col, int64_t N, int64_t s, int64_t nbn, int mode) {
  if (row >= N || row < col || col < s) return false;
  if (mode == 0) return true;
  if (mode == 4) return col >= s + nbn;
  return !(col < s + nbn && row < s + nbn);
}

__device__ __forceinline__ double lds_f64(unsigned addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ double dneg(double v) {   // exact sign flip on the integer pipe (not DADD)
  double r;
  asm("{\n .reg .b64 t;\n mov.b64 t, %1;\n xor.b64 t, t, 0x8000000000000000;\n mov.b64 %0, t;\n}\n"
      : "=d"(r) : "d"(v));
  return r;
}

__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap* map, int c0, int c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];\n" ::"l"(map), "r"(c0), "r"(c1) : "memory");
}
__device__ __forceinline__ void tma_reduce_add_2d(const CUtensorMap* map, int c0, int c1, unsigned src) {
  asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%1, %2}], [%3];\n" ::"l"(map),
               "r"(c0), "r"(c1), "r"(src)
               : "memory");
}
// 3-D forms (batched factorization: the third coordinate is the scenario)
__device__ __forceinline__ void tma_load_3d(unsigned dst, const CUtensorMap* map, int c0, int c1, int c2, unsigned bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(dst),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tma_prefetch_3d(const CUtensorMap* map, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];\n" ::"l"(map), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
__device__ __forceinline__ void tma_reduce_add_3d(const CUtensorMap* map, int c0, int c1, int c2, unsigned src) {
  asm volatile("cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.tile.bulk_group [%0, {%1, %2, %3}], [%4];\n" ::"l"(map),
               "r"(c0), "r"(c1), "r"(c2), "r"(src)
               : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, int c0, int c1, int c2, unsigned src) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];\n" ::"l"(map), "r"(c0),
               "r"(c1), "r"(c2), "r"(src)
               : "memory");
}
__device__ __forceinline__ void sts_f64(unsigned addr, double v) {
  asm volatile("st.shared.f64 [%0], %1;\n" ::"r"(addr), "d"(v) : "memory");
}

// The update no longer reads C at all: each group computes P = L21 W21^T for
// its tile from zero, writes -P (0 where the tile must not change: rows < s,
// cols < s, upper triangle) into the stage it just consumed, and one thread
// issues a TMA REDUCE-ADD of that tile into M (SASS UTMAREDG: the
// read-modify-write happens in L2).  The stage is released to the producer
// once the TMA engine has read it.
template <int mode, bool OUTB>
__global__ void __launch_bounds__(TTHREADS, 1) k_update_tma(int64_t N, double* __restrict__ A, int64_t lda, FWork f,
                                                             const __grid_constant__ CUtensorMap mapA,
                                                             const __grid_constant__ CUtensorMap mapW,
                                                             const __grid_constant__ CUtensorMap mapL,
                                                             const __grid_constant__ CUtensorMap mapX, int sched,
                                                             int64_t bt_tiles, int64_t bt_n) {
  // mode 5 = mode 0 for a batch of bt_n scenarios (3-D tensor maps, third coordinate = scenario):
  // the claim counter runs over bt_n * bt_tiles slots, slot x = scenario x / bt_tiles, tile
  // x % bt_tiles of that scenario's own lower trailing tile set (slots past it are skipped)
  // mode 6 = the F2 tiles of panel pidx itself (W21 = A21 X, L21, colmax) for every scenario of a
  // batch: slot x = scenario x / bt_tiles, 64-row tile x % bt_tiles below that scenario's block
  constexpr bool BT = (mode == 5 || mode == 6);
  const bool snake = (sched & 2) != 0 && !BT;
  // (a no-op unless launched as a programmatic dependent: then the whole predecessor --
  //  the exact panel that wrote pinfo / abort -- has completed and flushed past this point)
  pdl_wait();
  FCtl* ctl = f.ctl;
  if (!BT && ctl->abort) return;
  const int2 pi = BT ? make_int2(0, 1) : f.pinfo[f.pidx];
  const int64_t k0 = pi.x;
  const int kb = pi.y;
  const int64_t s = BT ? 0 : k0 + kb;
  if (!BT && (kb <= 0 || (mode == 0 && N - s <= 0))) return;   // (look-ahead modes still copy the last panel)
  const int64_t b0 = s / UT;
  const int64_t nt = (N - s > 0) ? (N + UT - 1) / UT - b0 : 0;
  const int64_t ntiles = (nt > 0) ? upd_ntiles(nt, mode) : 0;
  const int64_t nbn = (N - s) < NB ? (N - s) : NB;
  const int64_t nbn0 = nbn;
  // mode 3 also runs the NEXT panel's F2 tiles (W21 = A21 X, rows >= s + nbn)
  // as soon as that panel's F1 has published X: claimed before any update
  // tile, never waited for (the leftovers are k_panel_trsm's).
  // (tiles on the absolute 64-row grid: TMA box starts stay 16-byte aligned; rows < s + nbn are masked)
  const int64_t f2r0 = s + nbn;
  const int64_t f2r00 = f2r0;
  const int64_t f2base = (f2r0 / UT) * UT;
  const int64_t nf2 = (mode == 3 && N > f2r0) ? (N + UT - 1) / UT - f2r0 / UT : 0;
  constexpr bool LA = (mode == 3 || mode == 4);   // look-ahead modes (also copy the panel: S tiles)
  if (!BT && (int64_t)blockIdx.x >= ntiles + nf2 + (LA ? (N + UT - 1) / UT - k0 / UT : 0)) return;
  // (mode 6 claims from the panel's F2 slot: the same panel's update launch uses slot 3q)
  unsigned long long* counter = f.ucount + 3 * f.pidx + (mode == 6 ? 2 : 0);
  const int64_t nT1 = (LA && nt > 0) ? upd_nt1(nt, mode) : 0;
  // mode 3 also copies this panel's D + L from Lb into M (64-row "S" tiles, queued after T1)
  const int64_t nS = LA ? (N + UT - 1) / UT - k0 / UT : 0;
  const int64_t nall = BT ? bt_n * bt_tiles : ntiles + nS;
  unsigned long long* f2counter = f.ucount + 3 * (f.pidx + 1) + 2;
  extern __shared__ unsigned char tsm_raw[];
  // all shared addresses as 32-bit shared-window offsets (keeps LDS, not generic LD)
  const unsigned tsm = (smem_u32(tsm_raw) + 1023u) & ~1023u;
  constexpr int TS = OUTB ? 2 : 3;
  const unsigned full0 = tsm + TSMAX * TSTAGEB, empty0 = full0 + 8 * TSMAX;
  volatile long long* stile = reinterpret_cast<volatile long long*>(tsm_raw + (empty0 + 8 * TSMAX - smem_u32(tsm_raw)));
  volatile long long* stile2 = stile + TSMAX;   // BT: (scenario << 32 | its trailing start s)
  const unsigned outb0 = tsm + 2 * TSTAGEB;   // OUTB: group g stages -P at outb0 + g * TOPB
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < TS; i++) { mbar_init(full0 + 8 * i, 1); mbar_init(empty0 + 8 * i, 1); }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (warp == 0) {
    // ---------------- producer: one lane claims tiles from the launch's counter (dynamic
    // scheduling: CTAs that start late, e.g. behind the panel kernels, just take fewer tiles)
    // and issues their TMA loads; -1 in a stage's tile slot ends its consumer group
    if (lane == 0) {
      if (LA) { UTRACE_MIN(f.pidx, 0); USM_START(f.pidx); }
      int ends = 0;
      const bool dyn = (sched & 1) == 0;
      unsigned long long xnext = dyn ? atom_add_u64(counter, 1ull) : blockIdx.x;   // claimed one tile ahead
      bool f2open = nf2 > 0, xready = false;
      for (int i = 0; ends < TNG; i++) {
        const int st = i % TS, u = i / TS;
        if (u > 0) mbar_wait(empty0 + 8 * st, (u - 1) & 1);
        const unsigned fb = full0 + 8 * st;
        const unsigned sL = tsm + st * TSTAGEB, sW = sL + TOPB;
        if (f2open && xnext >= (unsigned long long)nT1) {   // (never while holding an unissued T1 tile)
          if (!xready) xready = ld_acquire_u32(&ctl->xready) >= (unsigned)(f.pidx + 2);
          if (xready) {
            const unsigned long long x2 = atom_add_u64(f2counter, 1ull);
            if (x2 < (unsigned long long)nf2) {
              const int R0 = (int)(f2base + (int64_t)x2 * UT);
              // the rows' T1 tiles (this launch's update of the next panel's columns) must have landed;
              // they were all claimed before any other tile and their CTAs never wait, so this is bounded
              const int64_t rlast = ((int64_t)R0 + UT - 1 < N - 1) ? (int64_t)R0 + UT - 1 : N - 1;
              for (int64_t BI = R0 / UT; BI <= rlast / UT; BI++) {
                const unsigned want = (unsigned)(f.pidx + 1);
                while (ld_acquire_u32(&f.t1flag[2 * BI]) < want) __nanosleep(64);
                if (nt >= 2 && BI > b0)
                  while (ld_acquire_u32(&f.t1flag[2 * BI + 1]) < want) __nanosleep(64);
              }
              stile[st] = (long long)((0xfffffffeull << 32) | (unsigned)R0);   // C0 = -2: F2 tile
              asm volatile("fence.proxy.async.global;\n" ::: "memory");     // X was written by the generic proxy
              mbar_expect_tx(fb, TSTAGEB);
#pragma unroll
              for (int b = 0; b < 4; b++) {
                tma_load_2d(sL + b * TBOXB, &mapA, R0 + 16 * b, (int)s, fb);   // A21 (updated by U_next)
                tma_load_2d(sW + b * TBOXB, &mapX, 16 * b, 0, fb);            // L11^{-1}
              }
              continue;
            }
            f2open = false;
          }
        }
        if constexpr (BT) {
          // claim until a slot that holds a real tile of a live scenario, or the end
          bool got = false;
          while (xnext < (unsigned long long)nall) {
            const unsigned long long xc = xnext;
            xnext = atom_add_u64(counter, 1ull);
            const int64_t sc = (int64_t)(xc / (unsigned long long)bt_tiles);
            int64_t lt = (int64_t)(xc % (unsigned long long)bt_tiles);
            const size_t bo = (size_t)sc * f.bws;
            const FCtl* cs = reinterpret_cast<const FCtl*>(reinterpret_cast<const char*>(f.ctl) + bo);
            if (cs->abort) continue;
            if constexpr (mode == 5) {
              // the first sched >> 8 slots of a scenario are its S tiles: 64-row blocks of the
              // panel's D + L (Lb) copied into M (replaces a separate k_panel_store launch)
              const int64_t nSmax = (int64_t)(sched >> 8);
              if (lt < nSmax) {
                const int2 ps = reinterpret_cast<const int2*>(reinterpret_cast<const char*>(f.pinfo) + bo)[f.pidx];
                const int64_t k0s = ps.x;
                if (ps.y <= 0 || lt >= (N + UT - 1) / UT - k0s / UT) continue;
                const int R0 = (int)((k0s / UT + lt) * UT);
                stile[st] = (long long)((0xfffffffdull << 32) | (unsigned)R0);   // C0 = -3: S tile
                stile2[st] = (long long)(((unsigned long long)sc << 32) | (unsigned long long)k0s);
                mbar_expect_tx(fb, TOPB);
#pragma unroll
                for (int b = 0; b < 4; b++) tma_load_3d(sL + b * TBOXB, &mapL, R0 + 16 * b, 0, (int)sc, fb);
                got = true;
                break;
              }
              lt -= nSmax;
            }
            if constexpr (mode == 6) {
              const int nbps = cs->nbp;
              const int64_t k0s = cs->k0, rb = k0s + nbps;
              if (nbps == 0 || rb >= N) continue;
              if (lt >= (N + UT - 1) / UT - rb / UT) continue;
              const int R0 = (int)((rb / UT + lt) * UT);
              stile[st] = (long long)((0xfffffffeull << 32) | (unsigned)R0);   // C0 = -2: F2 tile
              stile2[st] = (long long)(((unsigned long long)sc << 32) | (unsigned long long)rb);
              mbar_expect_tx(fb, TSTAGEB);
#pragma unroll
              for (int b = 0; b < 4; b++) {
                tma_load_3d(sL + b * TBOXB, &mapA, R0 + 16 * b, (int)k0s, (int)sc, fb);   // A21
                tma_load_3d(sW + b * TBOXB, &mapX, 16 * b, 0, (int)sc, fb);             // X = L11^{-T}
              }
              got = true;
              break;
            }
            const int2 ps = reinterpret_cast<const int2*>(reinterpret_cast<const char*>(f.pinfo) + bo)[f.pidx];
            const int64_t ss = (int64_t)ps.x + ps.y;
            if (ps.y <= 0 || N - ss <= 0) continue;
            const int64_t sb0 = ss / UT, snt = (N + UT - 1) / UT - sb0;
            if (lt >= snt * (snt + 1) / 2) continue;
            int64_t bi, bj;
            tri_tile(lt, bi, bj);
            const int R0 = (int)((sb0 + bi) * UT), C0 = (int)((sb0 + bj) * UT);
            stile[st] = (long long)(((unsigned long long)(unsigned)C0 << 32) | (unsigned)R0);
            stile2[st] = (long long)(((unsigned long long)sc << 32) | (unsigned long long)ss);
            mbar_expect_tx(fb, TSTAGEB);
#pragma unroll
            for (int b = 0; b < 4; b++) {
              tma_load_3d(sL + b * TBOXB, &mapL, R0 + 16 * b, 0, (int)sc, fb);
              tma_load_3d(sW + b * TBOXB, &mapW, C0 + 16 * b, 0, (int)sc, fb);
            }
            if (sched & 8)
#pragma unroll
              for (int b = 0; b < 4; b++) tma_prefetch_3d(&mapA, R0 + 16 * b, C0, (int)sc);
            got = true;
            break;
          }
          if (!got) {
            stile[st] = -1;
            mbar_arrive(fb);
            ends++;
          }
          continue;
        }
        const unsigned long long xc = xnext;
        if (xc >= (unsigned long long)nall) {
          f2open = false;          // never wait for X: the rest of the F2 tiles go to k_panel_trsm
          stile[st] = -1;
          mbar_arrive(fb);
          ends++;
          continue;
        }
        int64_t x = (int64_t)xc;
        if (LA && x >= nT1 && x < nT1 + nS) {   // S tile: Lb rows -> M
          const int R0 = (int)((k0 / UT + (x - nT1)) * UT);
          stile[st] = (long long)((0xfffffffdull << 32) | (unsigned)R0);   // C0 = -3
          mbar_expect_tx(fb, TOPB);
#pragma unroll
          for (int b = 0; b < 4; b++) tma_load_2d(sL + b * TBOXB, &mapL, R0 + 16 * b, 0, fb);
          xnext = dyn ? atom_add_u64(counter, 1ull) : xnext + gridDim.x;
          continue;
        }
        if (LA && x >= nT1) {
          x -= nS;
          // the bulk of the tiles runs in alternating direction from panel to panel, so
          // a pass starts on the tiles the previous pass touched last (still in L2)
          if (snake && (f.pidx & 1)) x = nT1 + (ntiles - 1 - x);
        }
        int64_t bi, bj;
        upd_tile(x, nt, mode, bi, bj);
        const int R0 = (int)((b0 + bi) * UT), C0 = (int)((b0 + bj) * UT);
        stile[st] = (long long)(((unsigned long long)(unsigned)C0 << 32) | (unsigned)R0);   // tile origin for the consumers
        mbar_expect_tx(fb, TSTAGEB);
#pragma unroll
        for (int b = 0; b < 4; b++) {
          tma_load_2d(sL + b * TBOXB, &mapL, R0 + 16 * b, 0, fb);
          tma_load_2d(sW + b * TBOXB, &mapW, C0 + 16 * b, 0, fb);
        }
        // pull the C tile into L2 now, so that its reduce-add (a tile later) is an L2 hit
        // and does not hold the TMA unit for a DRAM round trip
        if (sched & 8)
#pragma unroll
          for (int b = 0; b < 4; b++) tma_prefetch_2d(&mapA, R0 + 16 * b, C0);
        xnext = dyn ? atom_add_u64(counter, 1ull) : xnext + gridDim.x;
      }
      // every tile of this CTA is claimed: the next kernel of the stream (the next
      // panel's exact step) may be scheduled now; it still waits for this grid's end
      pdl_trigger();
    }
    return;
  }
  // ---------------- consumers: group grp takes stages grp, grp+TNG, ...
  const int grp = (warp - 1) >> 2, wq = (warp - 1) & 3;
  const int wm = (wq >> 1) * 32, wn = (wq & 1) * 32;
  const int g = lane >> 2, q = lane & 3;
  const bool leader = (wq == 0 && lane == 0);
  for (int i = grp;; i += TNG) {
    const int st = i % TS, u = i / TS;
    mbar_wait(full0 + 8 * st, u & 1);
    const long long x = stile[st];
    if (x == -1) break;
    const int64_t R0 = (int64_t)(unsigned)(x & 0xffffffffll), C0 = (int64_t)(x >> 32);
    const long long x2 = BT ? stile2[st] : 0;
    const int bsc = (int)(x2 >> 32);                               // BT: scenario
    const int64_t sT = BT ? (int64_t)(x2 & 0xffffffffll) : s;     // its trailing start
    if ((LA || mode == 5) && C0 == -3) {
      // S tile: panel rows R0..R0+63 of D + L (columns < kb, on/below the diagonal) into M
      double* Ac = A;
      int64_t k0c = k0;
      int kbc = kb;
      if constexpr (mode == 5) {   // (batched: that scenario's matrix and panel)
        Ac = A + (int64_t)bsc * f.bms;
        k0c = sT;
        kbc = reinterpret_cast<const int2*>(reinterpret_cast<const char*>(f.pinfo) + (size_t)bsc * f.bws)[f.pidx].y;
      }
      const unsigned Lt = tsm + st * TSTAGEB;
      if (mode == 5 && kbc == NB && R0 >= k0c + NB - 1) {
        // a full block strictly below the diagonal block: one TMA store of the staged Lb rows
        // (same swizzled 16 x 64 boxes as the load) into M
        if (leader) {
#pragma unroll
          for (int b = 0; b < 4; b++) tma_store_3d(&mapA, (int)(R0 + 16 * b), (int)k0c, bsc, Lt + b * TBOXB);
          asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
          asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");   // stage read by the TMA unit
          mbar_arrive(empty0 + 8 * st);
        }
        continue;
      }
      const int tq = (int)threadIdx.x - 32 - grp * 128;   // 0..127 within the group
      const int i = tq & 63;
      const int64_t row = R0 + i;
#pragma unroll 4
      for (int c = tq >> 6; c < NB; c += 2) {
        const double v = lds_f64(Lt + tma_off(i, c));
        if (c < kbc && row < N && row >= k0c + c) Ac[row + (k0c + c) * lda] = v;
      }
      asm volatile("bar.sync %0, 128;\n" ::"r"(grp + 1) : "memory");
      if (leader) mbar_arrive(empty0 + 8 * st);
      continue;
    }
    // F2 tile: its panel's width and pivots d, loaded now so their latency hides behind the
    // k-loop instead of stalling the epilogue's reciprocals
    int nbf = 0;
    double dpre[4][2];
    if (mode == 6 && C0 == -2) {   // (not mode 3: the extra live registers cost the single-system update more)
      const size_t bo = (mode == 6) ? (size_t)bsc * f.bws : 0;
      const FCtl* cf = reinterpret_cast<const FCtl*>(reinterpret_cast<const char*>(f.ctl) + bo);
      nbf = (mode == 6) ? __ldcg(&cf->nbp) : (int)nbn0;
#pragma unroll
      for (int b = 0; b < 4; b++)
#pragma unroll
        for (int e = 0; e < 2; e++) {
          const int c = wn + 8 * b + 2 * q + e;
          dpre[b][e] = (c < nbf) ? __ldcg(&cf->d[c]) : 0.0;
        }
    }
    double acc[4][4][2];
#pragma unroll
    for (int a = 0; a < 4; a++)
#pragma unroll
      for (int b = 0; b < 4; b++) acc[a][b][0] = acc[a][b][1] = 0.0;
    const unsigned Lt = tsm + st * TSTAGEB;
    const unsigned Lb = Lt + (unsigned)(wm >> 4) * TBOXB;
    const unsigned Wb = Lt + TOPB + (unsigned)(wn >> 4) * TBOXB;
    // k-loop with register double-buffered fragments (loads of step t+1 overlap the DMMAs of step t)
    double a0[4], b0v[4], a1[4], b1v[4];
    // k-step ks, lane (g, q) reads k = t(ks, q): a permutation of 0..63 (the contraction
    // order is free) chosen so that lanes q = 0,1 and q = 2,3 land in opposite bank
    // halves under the 128-byte swizzle (bit 2 of t selects the half): 2 wavefronts per LDS.64
    auto frag = [&](int ks, double* av, double* bv) {
      const unsigned t = 8u * (unsigned)(ks >> 1) + 4u * (unsigned)(q >> 1) + 2u * (unsigned)(ks & 1) + (unsigned)(q & 1);
      const unsigned sw = (t & 7u) << 4;
      const unsigned o0 = (t * 128u + (unsigned)g * 8u) ^ sw, o1 = (t * 128u + 64u + (unsigned)g * 8u) ^ sw;
#pragma unroll
      for (int a = 0; a < 4; a++) av[a] = lds_f64(Lb + (unsigned)(a >> 1) * TBOXB + ((a & 1) ? o1 : o0));
#pragma unroll
      for (int b = 0; b < 4; b++) bv[b] = lds_f64(Wb + (unsigned)(b >> 1) * TBOXB + ((b & 1) ? o1 : o0));
    };
    frag(0, a0, b0v);
#pragma unroll 1
    for (int ks = 0; ks < NB / 4; ks += 2) {
      frag(ks + 1, a1, b1v);
#pragma unroll
      for (int a = 0; a < 4; a++)
#pragma unroll
        for (int b = 0; b < 4; b++) dmma(acc[a][b][0], acc[a][b][1], a0[a], b0v[b]);
      if (ks + 2 < NB / 4) frag(ks + 2, a0, b0v);
#pragma unroll
      for (int a = 0; a < 4; a++)
#pragma unroll
        for (int b = 0; b < 4; b++) dmma(acc[a][b][0], acc[a][b][1], a1[a], b1v[b]);
    }
    // the whole group has finished reading L/W of this stage
    asm volatile("bar.sync %0, 128;\n" ::"r"(grp + 1) : "memory");
    if ((mode == 3 || mode == 6) && C0 == -2) {
      // F2 tile of the next panel (mode 6: of this panel, scenario bsc): W21 = acc,
      // L21 = acc D^{-1}, colmax (the stage is free already)
      if (leader) { mbar_arrive(empty0 + 8 * st); UTRACE_ADD(f.pidx, 2); }
      // (scenario bsc's control block and panel buffers by explicit byte offsets)
      const size_t bo = (mode == 6) ? (size_t)bsc * f.bws : 0;
      FCtl* cf = reinterpret_cast<FCtl*>(reinterpret_cast<char*>(f.ctl) + bo);
      const int64_t f2rf = (mode == 6) ? sT : f2r00;
      if (mode == 3) nbf = (int)nbn0;
      double* W2 = (mode == 6) ? reinterpret_cast<double*>(reinterpret_cast<char*>(f.W) + bo) : const_cast<double*>(f.Wprev);
      double* L2 = (mode == 6) ? reinterpret_cast<double*>(reinterpret_cast<char*>(f.Lb) + bo) : const_cast<double*>(f.Lbprev);
      double cm[4][2];
#pragma unroll
      for (int b = 0; b < 4; b++)
#pragma unroll
        for (int e = 0; e < 2; e++) {
          const int c = wn + 8 * b + 2 * q + e;
          const double d = (mode == 6) ? dpre[b][e] : ((c < nbf) ? __ldcg(&cf->d[c]) : 0.0);
          const double rd = fast_rcp(d);
          const double r1 = (d != 0.0) ? rd : 0.0;
          cm[b][e] = 0.0;
#pragma unroll
          for (int a = 0; a < 4; a++) {
            const int64_t row = R0 + wm + 8 * a + g;
            if (row < N && row >= f2rf && c < nbf) {
              W2[row + c * f.ldw] = acc[a][b][e];
              L2[row + c * f.ldw] = acc[a][b][e] * r1;
              cm[b][e] = fmax(cm[b][e], fabs(acc[a][b][e]));
            }
          }
          double v = cm[b][e];
          v = fmax(v, __shfl_xor_sync(0xffffffffu, v, 4));
          v = fmax(v, __shfl_xor_sync(0xffffffffu, v, 8));
          v = fmax(v, __shfl_xor_sync(0xffffffffu, v, 16));
          if (g == 0 && c < nbf) atomicMax(&cf->colmax[c], dbits(v));
        }
      continue;
    }
    // -P (masked) into the staging tile (OUTB: the group's own buffer, once its previous reduce has
    // read it, and the stage is released now; else the stage's L area), same swizzled box layout
    unsigned Ot = Lt;
    if (OUTB) {
      Ot = outb0 + (unsigned)grp * TOPB;
      if (leader) {
        mbar_arrive(empty0 + 8 * st);
        asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
      }
      asm volatile("bar.sync %0, 128;\n" ::"r"(grp + 1) : "memory");
    }
#pragma unroll
    for (int a = 0; a < 4; a++) {
      const int64_t row = R0 + wm + 8 * a + g;
#pragma unroll
      for (int b = 0; b < 4; b++)
#pragma unroll
        for (int e = 0; e < 2; e++) {
          const int cl = wn + 8 * b + 2 * q + e;
          const int64_t col = C0 + cl;
          const bool upd = upd_mask(row, col, N, sT, nbn, BT ? 0 : mode) && col >= sT;
          sts_f64(Ot + tma_off(wm + 8 * a + g, cl), upd ? dneg(acc[a][b][e]) : 0.0);
        }
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    asm volatile("bar.sync %0, 128;\n" ::"r"(grp + 1) : "memory");
    if (leader) {
#pragma unroll
      for (int b = 0; b < 4; b++) {
        if constexpr (BT) tma_reduce_add_3d(&mapA, (int)(R0 + 16 * b), (int)C0, bsc, Ot + b * TBOXB);
        else tma_reduce_add_2d(&mapA, (int)(R0 + 16 * b), (int)C0, Ot + b * TBOXB);
      }
      asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
      if (!OUTB) {
        asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");   // smem source consumed
        mbar_arrive(empty0 + 8 * st);
      }
      if (mode == 3 && C0 < (b0 + 2) * UT && nf2 > 0) {
        // T1 tile: publish its completion to the F2 tiles of the next panel
        asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
        asm volatile("fence.proxy.async.global;\n" ::: "memory");
        __threadfence();
        st_release_u32(&f.t1flag[2 * (R0 / UT) + (C0 / UT - b0)], (unsigned)(f.pidx + 1));
      }
    }
  }
  if (leader) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");   // reductions complete before exit
  if (LA && leader) { UTRACE_MAX(f.pidx, 1); USM_END(f.pidx); }
}

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                     const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                     CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

PFN_encodeTiled get_encode() {
  static const PFN_encodeTiled fn = []() -> PFN_encodeTiled {   // thread-safe one-time lookup
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    PFN_encodeTiled r = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      r = reinterpret_cast<PFN_encodeTiled>(p);
    (void)cudaGetLastError();
    return r;
  }();
  return fn;
}

// 2-D map over a column-major (rows x cols, ld) FP64 matrix; box 16 rows x 64 cols, 128-byte swizzle
bool make_map(CUtensorMap* m, const double* base, int64_t rows, int64_t cols, int64_t ld) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)rows, (cuuint64_t)cols};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 8};
  cuuint32_t box[2] = {16, 64};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace
#include "ozaki.cuh"
namespace {
// ---------------------------------------------------------------------------
// Finalize: inertia out; convert panel-end-order L to the explicit permutation
// form by applying every later panel's interchanges to earlier panels' rows
// (only if any interchange happened); final permutation + 2x2 flags into piv[N..2N).
// BLOCK = false: one cooperative grid for one system (grid.sync between phases);
// BLOCK = true: batched, one CTA per scenario (blockIdx.x), __syncthreads between phases.
template <bool BLOCK>
__device__ __forceinline__ void finalize_body(int64_t N, double* __restrict__ A, int64_t lda, FWork f, int32_t* piv,
                                              mds_inertia* inertia_out) {
  auto gsync = [] {
    if constexpr (BLOCK) __syncthreads();
    else cg::this_grid().sync();
  };
  FCtl* ctl = f.ctl;
  if (ctl->abort == 2) return;   // batched: scenario not re-factored this call (outputs kept)
  const int64_t gtid = BLOCK ? (int64_t)threadIdx.x : blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t gth = BLOCK ? (int64_t)blockDim.x : (int64_t)gridDim.x * blockDim.x;
  if (gtid == 0 && inertia_out) {
    inertia_out->pos = ctl->inertia[0];
    inertia_out->zero = ctl->inertia[1];
    inertia_out->neg = ctl->inertia[2];
  }
  if (ctl->abort) {
    // nothing was factored (non-finite input): leave a valid identity permutation with
    // 1x1 blocks so that a solve issued without looking at the status (a captured
    // graph) reads only in-range indices; its result is NaN and the status says why
    for (int64_t i = gtid; i < N; i += gth) piv[N + i] = (int)i;
    return;
  }
  for (int64_t i = gtid; i < N; i += gth) { f.rho[i] = (int)i; f.rhoinv[i] = (int)i; }
  const int npan = ctl->npanel;
  const int nswap = ctl->nswap;
  gsync();
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
        gsync();
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
      gsync();
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

__global__ void k_factor_finalize(int64_t N, double* __restrict__ A, int64_t lda, FWork f, int32_t* piv,
                                  mds_inertia* inertia_out) {
  finalize_body<false>(N, A, lda, f, piv, inertia_out);
}
__global__ void __launch_bounds__(512) k_factor_finalize_b(int64_t N, double* __restrict__ A, int64_t lda, FWork f,
                                                            int32_t* piv, mds_inertia* inertia_out) {
  bsel_ws(f, blockIdx.x);
  A += blockIdx.x * f.bms;
  piv += blockIdx.x * f.bps;
  finalize_body<true>(N, A, lda, f, piv, inertia_out ? inertia_out + blockIdx.x : nullptr);
}
}  // namespace

extern "C" int64_t mds_factor_panels(const void* fwork, int64_t N, int32_t* starts_host, int64_t cap) {
  if (!fwork || N <= 0) return MDS_ERR_ARG;
  FWork f = carve(const_cast<void*>(fwork), N, nullptr);
  FCtl c;
  if (cudaMemcpy(&c, f.ctl, sizeof(FCtl), cudaMemcpyDeviceToHost) != cudaSuccess) return MDS_ERR_CUDA;
  int64_t n = c.npanel;
  if (starts_host && cap > 0) {
    if (cudaMemcpy(starts_host, f.panel_start, sizeof(int32_t) * std::min<int64_t>(n, cap), cudaMemcpyDeviceToHost) !=
        cudaSuccess)
      return MDS_ERR_CUDA;
  }
  return n;
}

// Optional cap on the CTAs of the persistent update kernels (0 = all SMs);
// lets several factorizations on different streams share the GPU.
static int g_grid_cap = 0;
extern "C" int mds_factor_set_grid_cap(int ctas) {
  if (ctas < 0) return MDS_ERR_ARG;
  g_grid_cap = ctas;
  return MDS_OK;
}

// read by solve.cu
double* mds_factor_tol_ptr(const void* fwork) {
  return fwork ? &reinterpret_cast<FCtl*>(const_cast<void*>(fwork))->tol : nullptr;
}

// panels, interchanges and exact-path columns of the last mds_factor on `fwork` (synchronous)
extern "C" int mds_factor_stats(const void* fwork, int64_t* out4) {
  if (!fwork || !out4) return MDS_ERR_ARG;
  FCtl c;
  if (cudaMemcpy(&c, fwork, sizeof(FCtl), cudaMemcpyDeviceToHost) != cudaSuccess) return MDS_ERR_CUDA;
  out4[0] = c.npanel; out4[1] = c.nswap; out4[2] = c.nexact; out4[3] = c.abort;
  return MDS_OK;
}

// ||M||_inf and the zero-pivot tolerance the last mds_factor on `fwork` used (synchronous)
extern "C" int mds_factor_tol(const void* fwork, double* anorm_host, double* tol_host) {
  if (!fwork) return MDS_ERR_ARG;
  FCtl c;
  if (cudaMemcpy(&c, fwork, sizeof(FCtl), cudaMemcpyDeviceToHost) != cudaSuccess) return MDS_ERR_CUDA;
  if (anorm_host) *anorm_host = c.anorm;
  if (tol_host) *tol_host = c.tol;
  return MDS_OK;
}

// Side stream + reusable events for the look-ahead split, one set per CALLER
// stream (so concurrent factorizations on different streams never share
// events; a call on stream s always orders its side work through s).
struct LookaheadCtx {
  cudaStream_t side = nullptr;    // trailing updates
  std::vector<cudaEvent_t> ev;
};
static std::mutex g_la_mu;
static std::map<std::pair<int, cudaStream_t>, LookaheadCtx*> g_la;

static LookaheadCtx* lookahead_ctx(cudaStream_t st, size_t nev) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  std::lock_guard<std::mutex> lk(g_la_mu);
  LookaheadCtx*& c = g_la[std::make_pair(dev, st)];
  if (!c) {
    c = new LookaheadCtx();
    if (cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking) != cudaSuccess) {
      delete c;
      c = nullptr;
      return nullptr;
    }
  }
  while (c->ev.size() < nev) {
    cudaEvent_t e;
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return nullptr;
    c->ev.push_back(e);
  }
  return c;
}

extern "C" size_t mds_factor_workspace_size(int64_t N) {
  size_t total = 0;
  carve(nullptr, std::max<int64_t>(N, 1), &total);
  return total;
}

extern "C" int mds_factor(int64_t N, double* M, int64_t ldm, int32_t* piv, double zero_tol,
                          const double* anorm, mds_inertia* inertia_dev, mds_inertia* inertia_host, int32_t* status,
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
  // zero control + arrays (sw = -1); take ||M||_inf from the caller, or scan M for it
  MDS_LAUNCH(PC_ANORM, st,
             MDS_CUDA_TRY(launch_pdl(k_factor_init, dim3((unsigned)std::min<int64_t>(mds_cdiv(3 * (N + 2), 256), 1184)),
                                     dim3(256), 0, st, N, f, zero_tol, anorm, status, (const int32_t*)nullptr)));
  if (!anorm) {
    const int64_t nt = anorm::ntiles(N);
    MDS_LAUNCH(PC_ANORM, st,
               MDS_CUDA_TRY(launch_pdl(anorm::k_anorm_scan, dim3((unsigned)nt), dim3(256), 0, st, N, (const double*)M, ldm,
                                       (int64_t)0, f.nparts, (size_t)0)));
    anorm::NormOut o = {};
    o.anorm = &f.ctl->anorm;
    o.tol0 = &f.ctl->tol;
    o.abort0 = &f.ctl->abort;
    o.status = status;
    o.zero_tol = zero_tol;
    MDS_LAUNCH(PC_ANORM, st,
               MDS_CUDA_TRY(anorm::launch_rows(N, f.nparts, (size_t)0, o, 1, st)));
  }
  if (mds_once_per_device((const void*)k_update_tma<0, true>)) {
    cudaFuncSetAttribute(k_update_tma<0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, TSMEM);
    cudaFuncSetAttribute(k_update_tma<0, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, TSMEM);
    cudaFuncSetAttribute(k_update_tma<3, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, TSMEM);
    cudaFuncSetAttribute(k_update_tma<4, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, TSMEM);
    cudaFuncSetAttribute(k_panel_fast, cudaFuncAttributeMaxDynamicSharedMemorySize, F1SMEM);
    cudaFuncSetAttribute(k_update_tma<3, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, TSMEM);
    cudaFuncSetAttribute(k_panel_diag, cudaFuncAttributeMaxDynamicSharedMemorySize, F1SMEM);
    cudaFuncSetAttribute(k_panel_trsm, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * NB * US * (int)sizeof(double));
    cudaFuncSetAttribute(k_update<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * USTAGE * (int)sizeof(double));
    cudaFuncSetAttribute(k_update<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * USTAGE * (int)sizeof(double));
  }
  // 16-byte cp.async path needs a 16-byte aligned M, even ldm and a 16-byte aligned W
  const bool v16 = ((reinterpret_cast<uintptr_t>(M) & 15) == 0) && (ldm % 2 == 0) &&
                   ((reinterpret_cast<uintptr_t>(f.W) & 15) == 0);
  CUtensorMap mapA, mapW;
  const bool use_tma = v16 && !g_mds_var.no_tma && make_map(&mapA, M, N, N, ldm) &&
                       make_map(&mapW, f.W, N, NB, f.ldw);
  int sms = 148;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int64_t npmax = (N + (NB - 2)) / (NB - 1) + 1;
  // Look-ahead (TMA path).  Panel p's trailing update U(p) runs on a side
  // stream on all SMs but one, its dynamic tile queue starting with panel
  // p+1's columns.  Panel p+1's F1 applies panel p's update to its own
  // diagonal block, so it starts right after panel p's exact step,
  // concurrently with U(p); once F1 has published X, U(p)'s CTAs take panel
  // p+1's F2 tiles before any further update tile, and k_panel_trsm (after
  // U(p)) does whatever is left.  F4 (which may interchange anywhere) runs
  // after U(p).  U(p) also copies panel p's D + L from Lb into M (S tiles).
  const bool lookahead = use_tma && !g_mds_var.no_lookahead;
  constexpr int EVP = 2;   // events per panel: F4 done, U done
  cudaStream_t side = nullptr;
  std::vector<cudaEvent_t>* evs = nullptr;
  if (lookahead) {
    LookaheadCtx* c = lookahead_ctx(st, EVP * (size_t)npmax + EVP);
    if (!c) return MDS_ERR_CUDA;
    side = c->side;
    evs = &c->ev;
  }
  auto ev = [&](int64_t p, int k) { return (*evs)[EVP * p + k]; };
  CUtensorMap mapW1, mapL0, mapL1, mapX;
  if (use_tma && !(make_map(&mapW1, f.W1, N, NB, f.ldw) && make_map(&mapL0, f.Lb, N, NB, f.ldw) &&
                   make_map(&mapL1, f.Lb1, N, NB, f.ldw) && make_map(&mapX, f.Lblk, NB, NB, NB)))
    return MDS_ERR_CUDA;
  CUtensorMap mapOL, mapOW, mapOC;
  if (use_tma && g_mds_var.ozaki) {
    if (!(make_map_oz(&mapOL, f.ozL, N, 1, 0, OZ_TM) && make_map_oz(&mapOW, f.ozW, N, 1, 0, OZ_TN) &&
          make_map_ozc(&mapOC, M, N, ldm, 1, (size_t)ldm * N * 8)))
      return MDS_ERR_CUDA;
    if (mds_once_per_device((const void*)k_update_oz<false>)) {
      cudaFuncSetAttribute(k_update_oz<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, OZ_SMEM2);
      cudaFuncSetAttribute(k_update_oz<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, OZ_SMEM2);
    }
  }
  const int g_sched = (g_mds_var.static_sched ? 1 : 0) | (g_mds_var.no_snake ? 0 : 2) | (g_mds_var.no_cprefetch ? 0 : 8);
  const bool g_inplace = g_mds_var.upd_inplace != 0;
  const bool upd_main = g_mds_var.upd_main != 0;   // measured slower (A/B), off by default
  // panels with at most this many remaining rows use the one-launch fast path
  const bool capped = (g_grid_cap > 0 && g_grid_cap < sms);
  // (not when factorizations run concurrently (grid cap set): the tail launch's F2-role CTAs
  //  spin for X while F1 runs, which is free on an idle GPU but starves the other streams --
  //  C4: 3278 -> 4022 scenario-steps/s without it)
  const int64_t tail_rows = g_mds_var.tail_rows >= 0 ? (int64_t)g_mds_var.tail_rows : (capped ? 0 : 3500);
  if (capped) sms = g_grid_cap;
  const size_t usmem = 2 * NB * US * sizeof(double);
  auto fwork_for = [&](int64_t p) {
    FWork fp = f;
    fp.pidx = (int)p;
    fp.fuse = lookahead ? 1 : 0;
    if (p & 1) { fp.W = f.W1; fp.Lb = f.Lb1; fp.Wprev = f.W; fp.Lbprev = f.Lb; }
    else { fp.Wprev = f.W1; fp.Lbprev = f.Lb1; }
    return fp;
  };
  auto rows_of = [&](int64_t p) { return N - std::min<int64_t>(p * (NB - 1), N); };   // upper bound
  const int reserve = capped ? std::max(1, sms / 8) : 1;   // SMs left to the panel chain (F1)
  // F4 (acceptance + exact BK columns): multi-CTA, ~256 rows per CTA, all CTAs co-resident
  const bool f4_one_cta = g_mds_var.slow_1cta != 0;   // A/B: the single-CTA k_panel_slow
  const bool f4_no_ls = g_mds_var.exact_no_ls != 0;   // A/B: L rows read from L2
  const bool no_f2fold = g_mds_var.f2_trsm != 0;       // A/B: leftover F2 tiles by k_panel_trsm
  static thread_local int cl_ok = -1;   // (per thread; the attribute calls are idempotent)
  if (mds_once_per_device((const void*)k_panel_exact<false>)) {
    cudaFuncSetAttribute(k_panel_exact<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, XLS_MAX);
    cudaFuncSetAttribute(k_panel_exact<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, XLS_MAX);
    cudaFuncSetAttribute(k_panel_exact<true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cl_ok = -1;
  }
  if (cl_ok < 0) {   // can a 16-CTA cluster with the full shared-memory request be resident?
    cudaLaunchConfig_t qc = {};
    qc.gridDim = dim3(XCL);
    qc.blockDim = dim3(XT);
    qc.dynamicSmemBytes = XLS_MAX;
    cudaLaunchAttribute qa[1];
    qa[0].id = cudaLaunchAttributeClusterDimension;
    qa[0].val.clusterDim.x = XCL; qa[0].val.clusterDim.y = 1; qa[0].val.clusterDim.z = 1;
    qc.attrs = qa;
    qc.numAttrs = 1;
    int ncl = 0;
    cl_ok = (cudaOccupancyMaxActiveClusters(&ncl, k_panel_exact<true>, &qc) == cudaSuccess && ncl > 0) ? 1 : 0;
    (void)cudaGetLastError();
  }
  auto launch_f4 = [&](const FWork& fp, int64_t rows, int f2left) -> int {
    if (f4_one_cta) {
      MDS_LAUNCH(PC_PANEL_SLOW, st, MDS_CUDA_TRY(launch_pdl(k_panel_slow, dim3(1), dim3(1024), 0, st, N, M, ldm, fp, piv)));
      return MDS_OK;
    }
    const int64_t xrows = std::max<long long>(32, g_mds_var.exact_rows);
    // one thread-block cluster when its <= 16 CTAs keep their L rows in shared memory
    // (cluster barrier instead of the global counter); not for concurrent factorizations
    const bool cl = cl_ok == 1 && !capped && !f4_no_ls && g_mds_var.exact_cluster &&
                    rows <= (int64_t)XCL * ((XLS_MAX / (NB * 8) - 8) / 32 * 32);
    const unsigned g = cl ? (unsigned)std::max<int64_t>(1, std::min<int64_t>(mds_cdiv(rows, xrows), XCL))
                          : (unsigned)std::max<int64_t>(1, std::min<int64_t>({mds_cdiv(rows, xrows), (int64_t)sms, (int64_t)XMAXG}));
    const int chunk = (int)(mds_cdiv(mds_cdiv(std::max<int64_t>(rows, 1), g), 32) * 32);
    const size_t lsb = (size_t)NB * (chunk + 8) * sizeof(double);
    // (not for concurrent factorizations: a large shared-memory request per CTA would compete
    //  with the other streams' kernels even when no column takes the exact path)
    const int use_ls = (lsb <= (size_t)XLS_MAX && !f4_no_ls && !capped) ? 1 : 0;
    const size_t dsm = std::max<size_t>(use_ls ? lsb : 0, f2left ? usmem : 0);
    if (cl && use_ls) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(g);
      cfg.blockDim = dim3(XT);
      cfg.dynamicSmemBytes = dsm;
      cfg.stream = st;
      cudaLaunchAttribute at[2];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = g; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[1].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at;
      cfg.numAttrs = g_mds_var.no_pdl ? 1 : 2;
      MDS_LAUNCH(PC_PANEL_SLOW, st, MDS_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_panel_exact<true>, N, M, ldm, fp, piv, chunk,
                                                                    use_ls, f2left)));
      return MDS_OK;
    }
    MDS_LAUNCH(PC_PANEL_SLOW, st, MDS_CUDA_TRY(launch_coop_pdl(k_panel_exact<false>, dim3(g), dim3(XT), dsm, st, N, M, ldm,
                                                               fp, piv, chunk, use_ls, f2left)));
    return MDS_OK;
  };
  if (lookahead) {
    // Stream roles.  Update-bound panels: U(p) runs on the main stream right after
    // F4(p) (no cross-stream hop on the critical path) and F1(p+1) on the side
    // stream; tail panels (chain-bound): F1+F2 of p+1 (k_panel_fast) on the main
    // stream right after F4(p), U(p) on the side stream.
    // ev(p, 0): F4(p) done; ev(p, 1): the side-stream work launched after F4(p) done.
    auto launch_fast = [&](int64_t p) {
      const FWork fp = fwork_for(p);
      const unsigned g64 = (unsigned)std::max<int64_t>(mds_cdiv(rows_of(p), UT), 1);
      const unsigned gf = (unsigned)(1 + std::max<int64_t>(1, std::min<int64_t>(g64, 4 * (int64_t)sms)));
      MDS_LAUNCH(PC_PANEL_DIAG, st, MDS_CUDA_TRY(launch_pdl_prio(k_panel_fast, dim3(gf), dim3(256), F1SMEM, st, chain_prio(), N, M, ldm, fp)));
      return MDS_OK;
    };
    int64_t p = 0;
    bool tail = rows_of(0) <= tail_rows;
    if (tail) {
      if (int rc = launch_fast(0)) return rc;
    } else {
      const FWork fp = fwork_for(0);
      MDS_LAUNCH(PC_PANEL_DIAG, st, MDS_CUDA_TRY(launch_pdl_prio(k_panel_diag, dim3(1), dim3(256), F1SMEM, st, chain_prio(), N, M, ldm, fp)));
    }
    for (;; p++) {
      const int64_t rows = rows_of(p);
      const FWork fp = fwork_for(p);
      // F2 tiles U(p-1) did not take: a separate k_panel_trsm for the first panel (no U before it),
      // else done inside k_panel_exact (one launch fewer on the U(p-1) -> U(p) hand-off)
      const bool trsm_launch = !tail && (p == 0 || f4_one_cta || no_f2fold || capped);
      if (!tail) {
        if (p > 0) MDS_CUDA_TRY(cudaStreamWaitEvent(st, ev(p - 1, 1), 0));   // F1(p) (or U(p-1)) on the side stream
        if (trsm_launch) {
          const unsigned g64 = (unsigned)std::max<int64_t>(mds_cdiv(rows, UT), 1);
          MDS_LAUNCH(PC_PANEL_TRSM, st, (k_panel_trsm<<<g64, 128, usmem, st>>>(N, M, ldm, fp)));
        }
      } else if (p > 0) {
        MDS_CUDA_TRY(cudaStreamWaitEvent(st, ev(p - 1, 1), 0));   // U(p-1) on the side stream
      }
      if (int rc = launch_f4(fp, rows, (!tail && !trsm_launch) ? 1 : 0)) return rc;
      MDS_CUDA_TRY(cudaEventRecord(ev(p, 0), st));
      const int64_t n2max = std::max<int64_t>(rows - 1, 0);
      const int64_t nt = mds_cdiv(n2max, UT) + 1;
      const unsigned gr = (unsigned)std::max<int64_t>(1, std::min<int64_t>(nt * (nt + 1) / 2 + 2 * nt, sms - reserve));
      const CUtensorMap& mw = (p & 1) ? mapW1 : mapW;
      const CUtensorMap& ml = (p & 1) ? mapL1 : mapL0;
      const bool last = rows_of(p + 1) <= 0;
      const bool next_tail = last || rows_of(p + 1) <= tail_rows;
      MDS_CUDA_TRY(cudaStreamWaitEvent(side, ev(p, 0), 0));
      if (next_tail) {
        MDS_LAUNCH(PC_UPDATE, side,
                   (k_update_tma<4, true><<<gr, TTHREADS, TSMEM, side>>>(N, M, ldm, fp, mapA, mw, ml, mapX, g_sched, 0ll, 0ll)));
        MDS_CUDA_TRY(cudaEventRecord(ev(p, 1), side));
        if (last) break;
        if (int rc = launch_fast(p + 1)) return rc;
      } else if (!upd_main) {   // (A/B variant: U on the side stream, F1 on the main stream)
        if (g_inplace)
          MDS_LAUNCH(PC_UPDATE, side,
                     (k_update_tma<3, false><<<gr, TTHREADS, TSMEM, side>>>(N, M, ldm, fp, mapA, mw, ml, mapX, g_sched, 0ll, 0ll)));
        else
          MDS_LAUNCH(PC_UPDATE, side,
                     (k_update_tma<3, true><<<gr, TTHREADS, TSMEM, side>>>(N, M, ldm, fp, mapA, mw, ml, mapX, g_sched, 0ll, 0ll)));
        MDS_CUDA_TRY(cudaEventRecord(ev(p, 1), side));
        const FWork fn = fwork_for(p + 1);
        MDS_LAUNCH(PC_PANEL_DIAG, st, MDS_CUDA_TRY(launch_pdl_prio(k_panel_diag, dim3(1), dim3(256), F1SMEM, st, chain_prio(), N, M, ldm, fn)));
      } else {
        const FWork fn = fwork_for(p + 1);
        MDS_LAUNCH(PC_PANEL_DIAG, side, (k_panel_diag<<<1, 256, F1SMEM, side>>>(N, M, ldm, fn)));
        MDS_CUDA_TRY(cudaEventRecord(ev(p, 1), side));
        // programmatic dependent of the exact panel (same stream): the CTAs are resident and
        // past their prologue when it ends
        if (g_inplace)
          MDS_LAUNCH(PC_UPDATE, st, MDS_CUDA_TRY(launch_pdl(k_update_tma<3, false>, dim3(gr), dim3(TTHREADS), TSMEM, st, N, M,
                                                            ldm, fp, mapA, mw, ml, mapX, g_sched, 0ll, 0ll)));
        else
          MDS_LAUNCH(PC_UPDATE, st, MDS_CUDA_TRY(launch_pdl(k_update_tma<3, true>, dim3(gr), dim3(TTHREADS), TSMEM, st, N, M,
                                                            ldm, fp, mapA, mw, ml, mapX, g_sched, 0ll, 0ll)));
      }
      tail = next_tail;
    }
    MDS_CUDA_TRY(cudaStreamWaitEvent(st, ev(p, 1), 0));
  } else {
    for (int64_t p = 0; p < npmax; p++) {
      const int64_t rows = rows_of(p);
      if (rows <= 0) break;
      const FWork fp = fwork_for(p);
      const unsigned g256 = (unsigned)std::max<int64_t>(mds_cdiv(rows, 256), 1);
      const unsigned g64 = (unsigned)std::max<int64_t>(mds_cdiv(rows, UT), 1);
      const int64_t n2max = std::max<int64_t>(rows - 1, 0);
      const int64_t nt = mds_cdiv(n2max, UT) + 1;
      MDS_LAUNCH(PC_PANEL_DIAG, st, (k_panel_diag<<<1, 256, F1SMEM, st>>>(N, M, ldm, fp)));
      MDS_LAUNCH(PC_PANEL_TRSM, st, (k_panel_trsm<<<g64, 128, usmem, st>>>(N, M, ldm, fp)));
      if (int rc = launch_f4(fp, rows, 0)) return rc;
      const CUtensorMap& mw = (p & 1) ? mapW1 : mapW;
      const CUtensorMap& ml = (p & 1) ? mapL1 : mapL0;
      MDS_LAUNCH(PC_PANEL_STORE, st, (k_panel_store<<<dim3(g256, 8), 256, 0, st>>>(N, M, ldm, fp)));
      if (n2max > 0 && use_tma && g_mds_var.ozaki) {
        const int64_t smin = std::min<int64_t>(N, (p + 1) * (NB - 1));
        const int64_t r_lo = (smin / OZ_TM) * OZ_TM;
        MDS_LAUNCH(PC_UPDATE, st, MDS_CUDA_TRY(launch_pdl(k_oz_split, dim3((unsigned)mds_cdiv(N - r_lo, 64), 2, 1),
                                                          dim3(256), 0, st, N, fp, r_lo)));
        const int64_t tbo = oz_tiles(N, smin);
        const unsigned go = (unsigned)std::max<int64_t>(1, std::min<int64_t>(tbo, (int64_t)sms));
        MDS_LAUNCH(PC_UPDATE, st, (k_update_oz<false><<<go, OZ_THREADS2, OZ_SMEM2, st>>>(N, fp, mapOL, mapOW, mapOC,
                                                                                         tbo, 1)));
      } else if (n2max > 0) {
        const unsigned ugrid = (unsigned)std::min<int64_t>(nt * (nt + 1) / 2, sms);
        if (use_tma && g_inplace)
          MDS_LAUNCH(PC_UPDATE, st,
                     (k_update_tma<0, false><<<ugrid, TTHREADS, TSMEM, st>>>(N, M, ldm, fp, mapA, mw, ml, mapX, g_sched, 0ll, 0ll)));
        else if (use_tma)
          MDS_LAUNCH(PC_UPDATE, st,
                     (k_update_tma<0, true><<<ugrid, TTHREADS, TSMEM, st>>>(N, M, ldm, fp, mapA, mw, ml, mapX, g_sched, 0ll, 0ll)));
        else if (v16)
          MDS_LAUNCH(PC_UPDATE, st,
                     (k_update<true><<<ugrid, 128, 2 * USTAGE * sizeof(double), st>>>(N, M, ldm, fp)));
        else
          MDS_LAUNCH(PC_UPDATE, st,
                     (k_update<false><<<ugrid, 128, 2 * USTAGE * sizeof(double), st>>>(N, M, ldm, fp)));
      }
    }
  }
  {
    int dev = 0, sms = 148, occ = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_factor_finalize, 256, 0);
    // cooperative grid (grid-stride loops): the whole GPU for a lone factorization (the
    // row-interchange pass moves O(N^2) data when pivoting is heavy), a small grid when
    // several factorizations share the GPU (grid cap set: SCOPF batches)
    int blocks = (g_grid_cap > 0) ? std::min(32, sms * std::max(1, std::min(occ, 2)))
                                  : sms * std::max(1, std::min(occ, 4));
    void* args[] = {&N, &M, &ldm, &f, &piv, &inertia_dev};
    MDS_LAUNCH(PC_FINALIZE, st,
               MDS_CUDA_TRY(cudaLaunchCooperativeKernel((void*)k_factor_finalize, blocks, 256, args, 0, st)));
  }
  if (inertia_host) {
    if (!inertia_dev) return MDS_ERR_ARG;
    MDS_CUDA_TRY(cudaMemcpyAsync(inertia_host, inertia_dev, sizeof(mds_inertia), cudaMemcpyDeviceToHost, st));
    MDS_CUDA_TRY(cudaStreamSynchronize(st));
  }
  return MDS_OK;
}

// ---------------------------------------------------------------------------
// Batched factorization (SCOPF scenario batches, SURVEY §8(b) "_batched"): the
// same Bunch-Kaufman panels for `batch` independent N x N systems, one launch
// per step for ALL scenarios (grid.y = scenario), in the non-look-ahead order
// F1 -> F2 -> F4 -> store -> update.  The batch supplies the parallelism:
// F1 / F4 run one CTA per scenario, F2 / store one grid row per scenario, and
// the DMMA trailing update is ONE persistent launch whose tile queue spans every
// scenario's lower trailing tiles (3-D TMA maps, third coordinate = scenario).
namespace {
// 3-D map over `batch` column-major (rows x cols, ld) FP64 matrices `bstride` bytes apart
bool make_map3(CUtensorMap* m, const double* base, int64_t rows, int64_t cols, int64_t ld, int64_t batch,
               size_t bstride) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[3] = {(cuuint64_t)rows, (cuuint64_t)cols, (cuuint64_t)batch};
  cuuint64_t strides[2] = {(cuuint64_t)ld * 8, (cuuint64_t)bstride};
  cuuint32_t box[3] = {16, 64, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}
size_t factor_ws_stride(int64_t N) { return align_up(mds_factor_workspace_size(N), 256); }
}  // namespace

// per-scenario factor workspace stride (read by solve.cu for the batched tolerance)
size_t mds_factor_ws_stride_bytes(int64_t N) { return factor_ws_stride(std::max<int64_t>(N, 1)); }

extern "C" size_t mds_factor_batched_workspace_size(int64_t N, int64_t batch) {
  if (batch < 1) return 0;
  return (size_t)batch * factor_ws_stride(std::max<int64_t>(N, 1));
}

extern "C" int mds_factor_batched(int64_t batch, int64_t N, double* M, int64_t ldm, int64_t str_M, int32_t* piv,
                                  int64_t str_piv, double zero_tol, const double* anorm, mds_inertia* inertia_dev,
                                  int32_t* status, const int32_t* active, void* work, size_t work_bytes,
                                  void* stream) {
  if (batch < 0 || N < 0 || N >= (1 << 29)) return MDS_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  if (batch == 0) return MDS_OK;
  if (!inertia_dev || !status) return MDS_ERR_ARG;
  if (N == 0) {
    MDS_CUDA_TRY(cudaMemsetAsync(inertia_dev, 0, sizeof(mds_inertia) * batch, st));
    return MDS_OK;
  }
  if (!M || !piv || ldm < N || str_M < ldm * N || str_piv < 2 * N) return MDS_ERR_ARG;
  if (active && !anorm) return MDS_ERR_ARG;   // masked calls take ||M||_inf from the (masked) condensation
  // the batched update is TMA-only: 16-byte aligned matrices, even ldm and stride
  if ((reinterpret_cast<uintptr_t>(M) & 15) || (ldm & 1) || (str_M & 1)) return MDS_ERR_ARG;
  const size_t ws = factor_ws_stride(N);
  if (!work || work_bytes < (size_t)batch * ws) return MDS_ERR_WORKSPACE;
  FWork f = carve(work, N, nullptr);
  f.bws = ws;
  f.bms = str_M;
  f.bps = str_piv;
  const unsigned nb = (unsigned)batch;
  MDS_LAUNCH(PC_ANORM, st,
             MDS_CUDA_TRY(launch_pdl(k_factor_init, dim3((unsigned)std::min<int64_t>(mds_cdiv(3 * (N + 2), 256), 64), nb),
                                     dim3(256), 0, st, N, f, zero_tol, anorm, status, active)));
  if (!anorm) {
    MDS_LAUNCH(PC_ANORM, st,
               MDS_CUDA_TRY(launch_pdl(anorm::k_anorm_scan, dim3((unsigned)anorm::ntiles(N), nb), dim3(256), 0, st, N,
                                       (const double*)M, ldm, str_M, f.nparts, ws)));
    anorm::NormOut o = {};
    o.tol0 = &f.ctl->tol;
    o.abort0 = &f.ctl->abort;
    o.ctl_stride = ws;
    o.status = status;
    o.status_stride = 1;
    o.zero_tol = zero_tol;
    MDS_LAUNCH(PC_ANORM, st, MDS_CUDA_TRY(anorm::launch_rows(N, f.nparts, ws, o, batch, st)));
  }
  if (mds_once_per_device((const void*)k_update_tma<5, true>)) {
    cudaFuncSetAttribute(k_update_tma<5, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, TSMEM);
    cudaFuncSetAttribute(k_update_tma<6, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, TSMEM);
    cudaFuncSetAttribute(k_panel_diag, cudaFuncAttributeMaxDynamicSharedMemorySize, F1SMEM);
    cudaFuncSetAttribute(k_panel_trsm, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * NB * US * (int)sizeof(double));
  }
  CUtensorMap mapOL, mapOW, mapOC;
  if (g_mds_var.ozaki) {
    if (!(make_map_oz(&mapOL, f.ozL, N, batch, ws, OZ_TM) && make_map_oz(&mapOW, f.ozW, N, batch, ws, OZ_TN) &&
          make_map_ozc(&mapOC, M, N, ldm, batch, (size_t)str_M * 8)))
      return MDS_ERR_CUDA;
    if (mds_once_per_device((const void*)k_update_oz<true>)) {
      cudaFuncSetAttribute(k_update_oz<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, OZ_SMEM2);
      cudaFuncSetAttribute(k_update_oz<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, OZ_SMEM2);
    }
  }
  CUtensorMap mapA, mapW0, mapW1, mapL0, mapL1, mapX;
  if (!(make_map3(&mapA, M, N, N, ldm, batch, (size_t)str_M * 8) && make_map3(&mapX, f.Lblk, NB, NB, NB, batch, ws) &&
        make_map3(&mapW0, f.W, N, NB, f.ldw, batch, ws) && make_map3(&mapW1, f.W1, N, NB, f.ldw, batch, ws) &&
        make_map3(&mapL0, f.Lb, N, NB, f.ldw, batch, ws) && make_map3(&mapL1, f.Lb1, N, NB, f.ldw, batch, ws)))
    return MDS_ERR_CUDA;
  int sms = 148;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int sched = (g_mds_var.no_cprefetch ? 0 : 8);
  const size_t usmem = 2 * NB * US * sizeof(double);
  const int64_t npmax = (N + (NB - 2)) / (NB - 1) + 1;
  for (int64_t p = 0; p < npmax; p++) {
    const int64_t rows = N - std::min<int64_t>(p * (NB - 1), N);   // upper bound on the rows left
    if (rows <= 0) break;
    FWork fp = f;
    fp.pidx = (int)p;
    fp.fuse = 0;
    if (p & 1) { fp.W = f.W1; fp.Lb = f.Lb1; fp.Wprev = f.W; fp.Lbprev = f.Lb; }
    else { fp.Wprev = f.W1; fp.Lbprev = f.Lb1; }
    const unsigned g64 = (unsigned)std::max<int64_t>(mds_cdiv(rows, UT), 1);
    const unsigned g256 = (unsigned)std::max<int64_t>(mds_cdiv(rows, 256), 1);
    MDS_LAUNCH(PC_PANEL_DIAG, st, (k_panel_diag<<<dim3(1, nb), 256, F1SMEM, st>>>(N, M, ldm, fp)));
    if (g_mds_var.f2_trsm) {   // A/B: F2 by k_panel_trsm (one grid row per scenario)
      MDS_LAUNCH(PC_PANEL_TRSM, st, (k_panel_trsm<<<dim3(g64, nb), 128, usmem, st>>>(N, M, ldm, fp)));
    } else {   // F2 of every scenario as one TMA-fed DMMA launch (slots: 64-row tiles below the block)
      const int64_t rbmin = std::min<int64_t>(N, p * (NB - 1) + NB);
      const int64_t nt2 = (N + UT - 1) / UT - rbmin / UT;
      if (N > rbmin && nt2 > 0) {
        const unsigned gr = (unsigned)std::max<int64_t>(1, std::min<int64_t>(nt2 * batch, sms));
        const CUtensorMap& mw = (p & 1) ? mapW1 : mapW0;
        MDS_LAUNCH(PC_PANEL_TRSM, st,
                   (k_update_tma<6, true><<<gr, TTHREADS, TSMEM, st>>>(N, M, ldm, fp, mapA, mw, mw, mapX, sched, nt2,
                                                                       batch)));
      }
    }
    // F4 on one CTA per scenario (rows in one chunk, L rows read through L2; no grid barrier partners)
    const int chunk = (int)(mds_cdiv(rows, 32) * 32);
    MDS_LAUNCH(PC_PANEL_SLOW, st,
               MDS_CUDA_TRY(launch_pdl(k_panel_exact<false>, dim3(1, nb), dim3(XT), 0, st, N, M, ldm, fp, piv, chunk, 0, 0)));
    // trailing update of every scenario: slots per scenario = the tile count for the smallest
    // possible trailing start (every panel before p+1 finished at least NB-1 columns); the DMMA
    // update also copies the panel into M (S tiles, the first nS slots of each scenario)
    const int64_t smin = std::min<int64_t>(N, (p + 1) * (NB - 1));
    const int64_t nt = (N + UT - 1) / UT - smin / UT;
    const bool fold_store = N - smin > 0 && nt > 0 && !g_mds_var.ozaki;
    if (!fold_store) MDS_LAUNCH(PC_PANEL_STORE, st, (k_panel_store<<<dim3(g256, 8, nb), 256, 0, st>>>(N, M, ldm, fp)));
    if (N - smin > 0 && nt > 0) {
      const int64_t nS = (N + UT - 1) / UT - (p * (NB - 1)) / UT;   // 64-row blocks of the panel (k0 >= p (NB-1))
      const int64_t tb = nt * (nt + 1) / 2 + nS;
      const unsigned gr = (unsigned)std::max<int64_t>(1, std::min<int64_t>(tb * batch, sms));
      const CUtensorMap& mw = (p & 1) ? mapW1 : mapW0;
      const CUtensorMap& ml = (p & 1) ? mapL1 : mapL0;
      if (g_mds_var.ozaki) {
        const int64_t r_lo = (smin / OZ_TM) * OZ_TM;
        MDS_LAUNCH(PC_UPDATE, st, MDS_CUDA_TRY(launch_pdl(k_oz_split, dim3((unsigned)mds_cdiv(N - r_lo, 64), 2, nb),
                                                          dim3(256), 0, st, N, fp, r_lo)));
        const int64_t tbo = oz_tiles(N, smin);
        const unsigned go = (unsigned)std::max<int64_t>(1, std::min<int64_t>(tbo * batch, (int64_t)sms));
        MDS_LAUNCH(PC_UPDATE, st, (k_update_oz<true><<<go, OZ_THREADS2, OZ_SMEM2, st>>>(N, fp, mapOL, mapOW, mapOC, tbo,
                                                                                        batch)));
      } else {
        MDS_LAUNCH(PC_UPDATE, st,
                   (k_update_tma<5, true><<<gr, TTHREADS, TSMEM, st>>>(N, M, ldm, fp, mapA, mw, ml, mapA,
                                                                       sched | (int)(nS << 8), tb, batch)));
      }
    }
  }
  MDS_LAUNCH(PC_FINALIZE, st, (k_factor_finalize_b<<<nb, 512, 0, st>>>(N, M, ldm, f, piv, inertia_dev)));
  return MDS_OK;
}
