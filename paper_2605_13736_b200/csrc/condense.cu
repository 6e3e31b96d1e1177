// condense.cu — mds_plan_* and mds_condense[_batched]: Eq.(5) -> Eq.(6) of
// PAPER.md (K3 "M := M + A D B^T"), fused over
// CSR instead of the paper's three triplet launches, with the
// pre-factor ||M||_inf scan fused into the stores.
//
// The sparsity pattern of J_s is fixed across IPM iterations, so everything
// that depends only on it is done ONCE in mds_plan_create:
//   * every product term of M_yy = -J_s^T diag(w) J_s is a PAIR (p, p') of
//     entries of one CSR row k (p' <= p, both columns of row k): it lands on
//     M(n_d + colidx[p], n_d + colidx[p']) and equals (val_p w_k) val_p';
//   * pairs are sorted by destination -- 64x64 tile of M, column in the tile,
//     row in the tile -- and, for one destination, by k;
//   * one 64-bit word per pair: p | (p - p') << 32 | row << 52 | col << 58.
// Per call (device, stream-ordered, two kernels + one for the norm):
//   k_condense_rows   one pass over the sparse variables (a1): q_k, w_k = 1/q_k,
//                     status on q_k <= 0, and per CSR entry Q[p] = (val_p w_k,
//                     val_p).
//   k_condense_diag   one warp per constraint column: the diagonal pairs p = p'
//                     of M_yy(c, c) and the rhs term (J_s^T (w . r_xs))_c.
//   k_condense_tiles  persistent CTAs take 64x64 tiles of lower M from a queue
//                     (heaviest first): the dense blocks are copied
//                     (H_dd + diag(sigma_d) + delta_w I, J_d), the M_yy tiles are
//                     initialised (-delta_c, -1/d_h) and then stream their sorted
//                     pair list: a warp reads 32 pair words (coalesced), gathers
//                     the two Q values, forms the products, sums each run of equal
//                     destination with a segmented shuffle tree and subtracts the
//                     run sum from the shared-memory tile (one fixed order per
//                     destination: deterministic, no atomics; the order differs
//                     from the elimination's one-variable-at-a-time sums only by
//                     rounding, reading R7/R8).
//                     The tile is stored once (coalesced) and its fixed-order
//                     row/column abs-sum partials are written for ||M||_inf.
//   anorm::k_anorm_rows  fixed-order row sums + max (anorm.cuh).
// Deterministic; no atomics on data.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <new>
#include <numeric>
#include <vector>

#include "anorm.cuh"
#include "common.cuh"

struct mds_plan {
  int64_t n_s, n_d, m_E, m_I, nnz;
  int32_t* rowptr;   // [n_s+1] device
  int32_t* colidx;   // [nnz]   device
  int32_t* tptr;     // [m+1]   constraint-major transpose: entries of column c (residual.cu)
  int2* tkp;         // [nnz]   (k, p | min(suffix,31) << 27)
  int32_t max_col_len;
  // condensation pair lists (see top of file)
  int64_t npairs, ntile, nitems;
  uint32_t nbuf;               // part buffers (64x64) of the split tiles
  unsigned long long* pairs;   // [npairs] off-diagonal pairs, by tile, then (column, row), then k
  uint32_t* toff;              // [ntile + 1] pair range of each tile
  uint32_t* pbase;             // [ntile] first part buffer of a split tile
  uint32_t* order;             // [ntile] (I << 16 | J), heaviest tiles first (batched calls)
  uint2* items;                // [nitems] (I << 16 | J, part << 16 | nparts), heaviest first (single system)
};

namespace {
constexpr int CT = anorm::AT;         // tile edge (64)
constexpr int CW = anorm::AW;         // warps per CTA (8)
constexpr int PAIR_SBITS = 20;        // p - p' < 2^20 (row length limit of the pair encoding)
constexpr int64_t PART = 16384;       // pairs per work item of a split tile (single-system calls)
}  // namespace

extern "C" const char* mds_version(void) { return "mds_b200 0.2 sm_100a"; }

extern "C" int mds_plan_create(int64_t n_s, int64_t n_d, int64_t m_E, int64_t m_I,
                               const int32_t* rowptr, const int32_t* colidx, mds_plan** out) {
  if (!out || n_s < 0 || n_d < 0 || m_E < 0 || m_I < 0) return MDS_ERR_ARG;
  if (n_s > 0 && (!rowptr)) return MDS_ERR_ARG;
  const int64_t m = m_E + m_I, N = n_d + m;
  if (N > (int64_t)1 << 22) return MDS_ERR_ARG;   // tile coordinates are 16-bit (64-blocks)
  int64_t nnz = n_s > 0 ? rowptr[n_s] : 0;
  if (n_s > 0 && rowptr[0] != 0) return MDS_ERR_PATTERN;
  if (nnz > 0 && !colidx) return MDS_ERR_ARG;
  if (nnz >= ((int64_t)1 << 27)) return MDS_ERR_ARG;   // packed transpose map limit
  // validate canonical CSR (reading R13): sorted, unique, in range
  int64_t maxrow = 0;
  for (int64_t k = 0; k < n_s; k++) {
    if (rowptr[k + 1] < rowptr[k]) return MDS_ERR_PATTERN;
    maxrow = std::max<int64_t>(maxrow, rowptr[k + 1] - rowptr[k]);
    for (int64_t p = rowptr[k]; p < rowptr[k + 1]; p++) {
      if (colidx[p] < 0 || colidx[p] >= m) return MDS_ERR_PATTERN;
      if (p > rowptr[k] && colidx[p] <= colidx[p - 1]) return MDS_ERR_PATTERN;
    }
  }
  if (maxrow >= ((int64_t)1 << PAIR_SBITS)) return MDS_ERR_ARG;
  // constraint-major transpose (counting sort; entries of a column in k order)
  std::vector<int32_t> tptr(m + 1, 0);
  for (int64_t p = 0; p < nnz; p++) tptr[colidx[p] + 1]++;
  for (int64_t c = 0; c < m; c++) tptr[c + 1] += tptr[c];
  std::vector<int2> tkp(std::max<int64_t>(nnz, 1));
  {
    std::vector<int32_t> fill(tptr.begin(), tptr.end() - 1);
    for (int64_t k = 0; k < n_s; k++)
      for (int64_t p = rowptr[k]; p < rowptr[k + 1]; p++) {
        const unsigned sl = (unsigned)std::min<int64_t>(rowptr[k + 1] - p, 31);
        tkp[fill[colidx[p]]++] = make_int2((int)k, (int)((unsigned)p | (sl << 27)));
      }
  }
  int32_t maxlen = 0;
  for (int64_t c = 0; c < m; c++) maxlen = std::max(maxlen, tptr[c + 1] - tptr[c]);

  // ---- condensation pair lists (off-diagonal pairs p' < p only: the diagonal
  //      pairs p = p' are summed per constraint column by k_condense_diag):
  //      counting sort by tile, then by (column, row) inside a tile, stable in k
  const int64_t nb = (N + CT - 1) / CT, ntile = anorm::ntiles(N);
  auto tile_of = [&](int64_t row, int64_t col) { return anorm::tile_id(row / CT, col / CT); };
  std::vector<int64_t> tcount(ntile + 1, 0);
  int64_t npairs = 0;
  for (int64_t k = 0; k < n_s; k++)
    for (int64_t p = rowptr[k]; p < rowptr[k + 1]; p++)
      for (int64_t pp = rowptr[k]; pp < p; pp++) {
        tcount[tile_of(n_d + colidx[p], n_d + colidx[pp]) + 1]++;
        npairs++;
      }
  if (npairs >= ((int64_t)1 << 32)) return MDS_ERR_ARG;
  for (int64_t t = 0; t < ntile; t++) tcount[t + 1] += tcount[t];
  std::vector<unsigned long long> pairs(std::max<int64_t>(npairs, 1));
  {
    std::vector<int64_t> fill(tcount.begin(), tcount.end() - 1);
    for (int64_t k = 0; k < n_s; k++)                                  // k ascending: stable by k
      for (int64_t p = rowptr[k]; p < rowptr[k + 1]; p++)
        for (int64_t pp = rowptr[k]; pp < p; pp++) {
          const int64_t row = n_d + colidx[p], col = n_d + colidx[pp];
          const unsigned long long w = (unsigned long long)(uint32_t)p |
                                       ((unsigned long long)(p - pp) << 32) |
                                       ((unsigned long long)(row % CT) << 52) |
                                       ((unsigned long long)(col % CT) << 58);
          pairs[fill[tile_of(row, col)]++] = w;
        }
  }
  {
    std::vector<unsigned long long> tmp;
    std::vector<int64_t> cnt(CT * CT + 1);
    for (int64_t t = 0; t < ntile; t++) {
      const int64_t a = tcount[t], b = tcount[t + 1];
      if (b - a < 2) continue;
      // stable counting sort of this tile's pairs by (col, row) = bits 52..63
      std::fill(cnt.begin(), cnt.end(), 0);
      auto key = [](unsigned long long w) { return (int)(w >> 52); };
      for (int64_t q = a; q < b; q++) cnt[key(pairs[q]) + 1]++;
      for (int i = 0; i < CT * CT; i++) cnt[i + 1] += cnt[i];
      tmp.assign(b - a, 0ull);
      for (int64_t q = a; q < b; q++) tmp[cnt[key(pairs[q])]++] = pairs[q];
      std::copy(tmp.begin(), tmp.end(), pairs.begin() + a);
    }
  }
  // Work items.  Every tile is one item for batched calls (the batch supplies the
  // parallelism).  For a single system, a tile with more than PART pairs is cut
  // into parts (chunk-aligned ranges of its list); each part sums into its own
  // buffer and the last part to finish merges them in part order.  Items are
  // processed heaviest first.
  std::vector<uint32_t> order;                 // tiles: (I << 16 | J)
  std::vector<uint2> items;                    // parts: (I << 16 | J, part << 16 | nparts)
  std::vector<uint32_t> pbase(ntile, 0);
  uint32_t nbuf = 0;
  {
    std::vector<std::pair<int64_t, uint32_t>> cost;
    std::vector<std::pair<int64_t, uint2>> icost;
    cost.reserve(ntile);
    for (int64_t I = 0; I < nb; I++)
      for (int64_t J = 0; J <= I; J++) {
        const int64_t t = anorm::tile_id(I, J), np_ = tcount[t + 1] - tcount[t];
        const uint32_t ij = (uint32_t)((I << 16) | J);
        cost.emplace_back(-(4 * np_ + CT * CT / 8), ij);
        const int64_t nparts = std::min<int64_t>(std::max<int64_t>(1, mds_cdiv(np_, PART)), 0xffff);
        if (nparts > 1) { pbase[t] = nbuf; nbuf += (uint32_t)nparts; }
        for (int64_t q = 0; q < nparts; q++)
          icost.emplace_back(-(4 * mds_cdiv(np_, nparts) + (nparts > 1 ? CT * CT / 4 : CT * CT / 8)),
                             make_uint2(ij, (uint32_t)((q << 16) | nparts)));
      }
    std::stable_sort(cost.begin(), cost.end(),
                     [](const std::pair<int64_t, uint32_t>& x, const std::pair<int64_t, uint32_t>& y) {
                       return x.first < y.first;
                     });
    std::stable_sort(icost.begin(), icost.end(),
                     [](const std::pair<int64_t, uint2>& x, const std::pair<int64_t, uint2>& y) {
                       return x.first < y.first;
                     });
    for (auto& c : cost) order.push_back(c.second);
    for (auto& c : icost) items.push_back(c.second);
  }
  std::vector<uint32_t> toff(ntile + 1);
  for (int64_t t = 0; t <= ntile; t++) toff[t] = (uint32_t)tcount[t];

  mds_plan* P = new (std::nothrow) mds_plan();
  if (!P) return MDS_ERR_ARG;
  P->n_s = n_s; P->n_d = n_d; P->m_E = m_E; P->m_I = m_I; P->nnz = nnz; P->max_col_len = maxlen;
  P->npairs = npairs; P->ntile = ntile; P->nitems = (int64_t)items.size(); P->nbuf = nbuf;
  P->rowptr = nullptr; P->colidx = nullptr; P->tptr = nullptr; P->tkp = nullptr;
  P->pairs = nullptr; P->toff = nullptr; P->pbase = nullptr; P->order = nullptr; P->items = nullptr;
  auto up = [](void** dst, const void* src, size_t bytes) {
    if (cudaMalloc(dst, std::max<size_t>(bytes, 16)) != cudaSuccess) return false;
    return bytes == 0 || cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice) == cudaSuccess;
  };
  std::vector<int32_t> rp(n_s + 1, 0);
  if (n_s > 0) std::memcpy(rp.data(), rowptr, sizeof(int32_t) * (n_s + 1));
  bool ok = up((void**)&P->rowptr, rp.data(), sizeof(int32_t) * (n_s + 1)) &&
            up((void**)&P->colidx, colidx, sizeof(int32_t) * nnz) &&
            up((void**)&P->tptr, tptr.data(), sizeof(int32_t) * (m + 1)) &&
            up((void**)&P->tkp, tkp.data(), sizeof(int2) * nnz) &&
            up((void**)&P->pairs, pairs.data(), sizeof(unsigned long long) * npairs) &&
            up((void**)&P->toff, toff.data(), sizeof(uint32_t) * (ntile + 1)) &&
            up((void**)&P->pbase, pbase.data(), sizeof(uint32_t) * ntile) &&
            up((void**)&P->order, order.data(), sizeof(uint32_t) * order.size()) &&
            up((void**)&P->items, items.data(), sizeof(uint2) * items.size());
  if (!ok) {
    mds_plan_destroy(P);
    return MDS_ERR_CUDA;
  }
  *out = P;
  return MDS_OK;
}

extern "C" int mds_plan_destroy(mds_plan* P) {
  if (!P) return MDS_ERR_ARG;
  cudaFree(P->rowptr); cudaFree(P->colidx); cudaFree(P->tptr); cudaFree(P->tkp);
  cudaFree(P->pairs); cudaFree(P->toff); cudaFree(P->pbase); cudaFree(P->order); cudaFree(P->items);
  delete P;
  return MDS_OK;
}

extern "C" int mds_plan_dims(const mds_plan* P, int64_t* out) {
  if (!P || !out) return MDS_ERR_ARG;
  out[0] = P->n_s; out[1] = P->n_d; out[2] = P->m_E; out[3] = P->m_I; out[4] = P->nnz;
  return MDS_OK;
}

// accessors for solve.cu / residual.cu (same library)
const int32_t* mds_plan_rowptr(const mds_plan* P) { return P->rowptr; }
const int32_t* mds_plan_colidx(const mds_plan* P) { return P->colidx; }
const int32_t* mds_plan_tptr(const mds_plan* P) { return P->tptr; }
const int2* mds_plan_tkp(const mds_plan* P) { return P->tkp; }

namespace {
// ---------------------------------------------------------------------------
// Per-call arguments.  Every per-scenario array is (base, stride in elements);
// the single-system call uses batch = 1 and strides 0.
struct CondArgs {
  int64_t n_s, n_d, m_E, m, N, nnz, ntile, nitems, batch;
  const int32_t* active;                // [batch] or NULL: scenarios with active[s] == 0 are left untouched
  const int32_t* rowptr;
  const int32_t* tptr;
  const int2* tkp;
  const unsigned long long* pairs;
  const uint32_t* toff;
  const uint32_t* pbase;
  const uint32_t* order;
  const uint2* items;
  int split;                            // 1: walk `items` (split tiles), 0: walk `order`
  const double* val; int64_t s_val;
  const double* h_ss; int64_t s_hss;
  const double* sigma_s; int64_t s_sig;
  const double* H; int64_t ldh, s_H;
  const double* sigma_d; int64_t s_sd;
  const double* Jd; int64_t ldj, s_J;
  const double* d_h; int64_t s_dh;
  double delta_w, delta_c;              // scalars, or per scenario from:
  const double* dw_arr; const double* dc_arr;
  const double* r; int64_t s_r;         // [n_s + N] per scenario, or NULL
  double* M; int64_t ldm, s_M;
  double* rhs; int64_t s_rhs;           // or NULL
  double* w; int64_t s_w;
  double* anorm;                        // [batch] or NULL
  int32_t* status; int64_t s_st;        // per-scenario status (stride 0: shared)
  // workspace
  double2* Q;        // [batch][nnz]  (val_p w_k, val_p)
  double* dsum;      // [batch][m]    sum over column c of val^2 w (the diagonal pairs)
  double* pbuf;      // [nbuf][64*64] part sums of split tiles
  unsigned* ticket;  // [ntile]       parts finished per split tile
  char* parts;       // [batch][parts_bytes(N)]
  size_t parts_stride;
  unsigned* queue;   // [4] tile queue counter
};

__device__ __forceinline__ anorm::Parts parts_of(const CondArgs& a, int64_t s) {
  return anorm::parts_at(a.parts + (size_t)s * a.parts_stride, a.N);
}

__device__ __forceinline__ unsigned long long pol_evict_last() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ unsigned long long pol_evict_first() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ double ld_d(const double* a, unsigned long long pol) {
  double v;
  asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ unsigned long long ld_pair(const unsigned long long* a, unsigned long long pol) {
  unsigned long long v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ void st_stream(double* a, double v) {   // streaming store (evict-first)
  asm volatile("st.global.cs.f64 [%0], %1;" ::"l"(a), "d"(v) : "memory");
}
__device__ __forceinline__ void st_keep2(double2* a, double2 v, unsigned long long pol) {
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(a), "d"(v.x), "d"(v.y), "l"(pol) : "memory");
}
__device__ __forceinline__ double2 ld_q(const double2* a, unsigned long long pol) {
  double2 v;
  asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(a), "l"(pol));
  return v;
}

// ---------------------------------------------------------------------------
// a1 + per-entry factors.  A warp takes 32 consecutive sparse variables: lane l
// forms q = (h_ss + sigma_s) + delta_w and w = 1/q of variable k0 + l (IEEE
// division, as the elimination), then the warp walks the entries of those 32
// rows (contiguous in CSR) with coalesced loads, finds each entry's row by a
// 5-step shuffle search over the row pointers and stores t_p = val_p w_k.
// Also zeroes the tile queue, the split-tile tickets and the norm counters.
__global__ void __launch_bounds__(256) k_condense_rows(CondArgs a) {
  pdl_wait();
  pdl_trigger();
  const int64_t gt = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (gt < 4) a.queue[gt] = 0u;
  if (a.split) for (int64_t i = gt; i < a.ntile; i += (int64_t)gridDim.x * blockDim.x) a.ticket[i] = 0u;
  if (a.anorm && gt < a.batch * 4) {
    anorm::Parts P = parts_of(a, gt / 4);
    P.ctr[gt % 4] = 0u;
  }
  const int lane = threadIdx.x & 31;
  const int64_t nblk = mds_cdiv(a.n_s, 32);
  const int64_t gw = gt >> 5, nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const unsigned long long pol_keep = pol_evict_last();
  for (int64_t g = gw; g < a.batch * nblk; g += nw) {
    const int64_t s = g / nblk, k0 = (g - s * nblk) * 32;
    if (a.active && !a.active[s]) continue;
    const int64_t k = k0 + lane;
    const int nrow = (int)min((int64_t)32, a.n_s - k0);
    double wk = 0.0;
    int rp = 0;
    if (lane < nrow) {
      const double dw = a.dw_arr ? a.dw_arr[s] : a.delta_w;
      const double q = __dadd_rn(__dadd_rn(a.h_ss[s * a.s_hss + k], a.sigma_s[s * a.s_sig + k]), dw);
      if (!(q > 0.0)) mds_set_status(a.status + s * a.s_st, MDS_ERR_NONPOSITIVE);
      wk = 1.0 / q;
      a.w[s * a.s_w + k] = wk;
      rp = a.rowptr[k];
    }
    const int p0 = __shfl_sync(0xffffffffu, rp, 0);
    const int p1 = a.rowptr[k0 + nrow];
    const double* val = a.val + s * a.s_val;
    double2* Q = a.Q + s * a.nnz;
    for (int p = p0 + lane; __any_sync(0xffffffffu, p < p1); p += 32) {
      // largest row r < nrow with rowptr[k0 + r] <= p (rows may be empty)
      int lo = 0;
#pragma unroll
      for (int step = 16; step >= 1; step >>= 1) {
        const int cand = lo + step;
        const int rc = __shfl_sync(0xffffffffu, rp, cand < nrow ? cand : 0);
        if (cand < nrow && rc <= p) lo = cand;
      }
      const double wr = __shfl_sync(0xffffffffu, wk, lo);
      if (p < p1) {
        const double v = val[p];
        st_keep2(Q + p, make_double2(__dmul_rn(v, wr), v), pol_keep);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// The diagonal pairs and the right-hand side, one warp per constraint column c
// (its entries in k order from the plan's transpose): dsum[c] = sum over the
// column of t_p val_p (the p = p' products of M_yy(c, c)), and
// rhs_c = [r_xd; r_y - J_s^T (w . r_xs)] with the column sum of t_p r_xs[k].
// Lane-strided partial sums in a fixed order, then a fixed warp tree.
__global__ void __launch_bounds__(256) k_condense_diag(CondArgs a) {
  pdl_wait();
  pdl_trigger();
  const int lane = threadIdx.x & 31;
  const int64_t s = blockIdx.y;
  if (a.active && !a.active[s]) return;
  const int64_t c = blockIdx.x * 8ll + (threadIdx.x >> 5);
  const double* r = a.r ? a.r + s * a.s_r : nullptr;
  double* rhs = (a.rhs && r) ? a.rhs + s * a.s_rhs : nullptr;
  if (rhs) {
    for (int64_t j = blockIdx.x * 256ll + threadIdx.x; j < a.n_d; j += (int64_t)gridDim.x * 256)
      rhs[j] = r[a.n_s + j];
  }
  if (c >= a.m) return;
  const double2* Q = a.Q + s * a.nnz;
  const unsigned long long pol_keep = pol_evict_last();
  const int e0 = a.tptr[c], e1 = a.tptr[c + 1];
  constexpr int U = 4;               // independent entries in flight per lane
  double sd[U], sr[U];
#pragma unroll
  for (int u = 0; u < U; u++) sd[u] = sr[u] = 0.0;
  for (int e = e0 + lane; e < e1; e += 32 * U) {
    int2 kp[U];
#pragma unroll
    for (int u = 0; u < U; u++) kp[u] = (e + 32 * u < e1) ? a.tkp[e + 32 * u] : make_int2(-1, 0);
    double2 q[U];
    double rk[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      q[u] = make_double2(0.0, 0.0);
      rk[u] = 0.0;
      if (kp[u].x >= 0) {
        q[u] = ld_q(Q + (kp[u].y & ((1 << 27) - 1)), pol_keep);
        if (r) rk[u] = r[kp[u].x];
      }
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
      sd[u] += __dmul_rn(q[u].x, q[u].y);
      sr[u] += __dmul_rn(q[u].x, rk[u]);
    }
  }
  double d = (sd[0] + sd[1]) + (sd[2] + sd[3]), rr = (sr[0] + sr[1]) + (sr[2] + sr[3]);
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    d += __shfl_xor_sync(0xffffffffu, d, o);
    rr += __shfl_xor_sync(0xffffffffu, rr, o);
  }
  if (lane == 0) {
    a.dsum[s * a.m + c] = d;
    if (rhs) rhs[a.n_d + c] = __dsub_rn(r[a.n_s + a.n_d + c], rr);
  }
}

// Subtract the pair products of list range [r0, r1) (sorted by destination key
// = column << 6 | row) from the shared tile T.  One warp, 32 pairs per chunk,
// two chunks in flight; each run of equal destination inside a chunk is summed
// by a segmented shuffle tree and its last lane subtracts the run sum.  The
// range's first run, when it continues the pair before the range (ckey), is
// summed into the returned carry instead (the caller subtracts it later, in
// warp order).  *carried = its destination, or -1.
__device__ __forceinline__ double pair_range(const unsigned long long* __restrict__ pairs, uint32_t r0, uint32_t r1,
                                             int ckey, const double2* __restrict__ Q, double* T, int lane, unsigned long long pol_stream,
                                             unsigned long long pol_keep, int* carried) {
  double carry = 0.0;
  *carried = -1;
  for (uint32_t base = r0; base < r1; base += 64) {
    double prod[2];
    int key[2];
#pragma unroll
    for (int u = 0; u < 2; u++) {
      const uint32_t idx = base + 32 * u + lane;
      key[u] = 4096 + lane;   // invalid lanes: distinct keys that never match
      prod[u] = 0.0;
      if (idx < r1) {
        const unsigned long long wd = ld_pair(pairs + idx, pol_stream);
        const uint32_t p = (uint32_t)wd;
        const uint32_t sft = (uint32_t)(wd >> 32) & ((1u << PAIR_SBITS) - 1u);
        key[u] = (int)(wd >> 52);
        prod[u] = __dmul_rn(ld_q(Q + p, pol_keep).x, ld_q(Q + (p - sft), pol_keep).y);
      }
    }
#pragma unroll
    for (int u = 0; u < 2; u++) {
      if (base + 32 * u >= r1) break;
      double v = prod[u];
      const int k = key[u];
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const double o = __shfl_up_sync(0xffffffffu, v, d);
        const int ok = __shfl_up_sync(0xffffffffu, k, d);
        if (lane >= d && ok == k) v += o;
      }
      const int nk = __shfl_down_sync(0xffffffffu, k, 1);
      bool tail = (base + 32 * u + lane < r1) && (lane == 31 || nk != k);
      if (ckey >= 0) {   // still inside the run continued from before the range
        const int k0 = __shfl_sync(0xffffffffu, k, 0);
        if (k0 == ckey) {
          const unsigned same = __ballot_sync(0xffffffffu, k == ckey);
          const int tl = 31 - __clz(same);
          carry += __shfl_sync(0xffffffffu, v, tl);
          *carried = ckey;
          if (k == ckey) tail = false;
          if (tl < 31) ckey = -1;
        } else {
          ckey = -1;
        }
      }
      if (tail) T[(k >> 6) * CT + (k & 63)] -= v;
      __syncwarp();
    }
  }
  return carry;
}

// Initial value of lower M(i, j) before the off-diagonal pairs: the dense blocks of
// Eq.(6) (H_dd + diag(sigma_d) + delta_w I, J_d) or the M_yy diagonal start
// (-delta_c - 1/d_h - the diagonal pairs), 0 elsewhere (and outside the lower triangle).
__device__ __forceinline__ double init_value(const CondArgs& a, int64_t s, int64_t i, int64_t j, double dw, double dc,
                                            unsigned long long pol_stream) {
  const int64_t n_d = a.n_d, N = a.N;
  double v = 0.0;
  if (i < N && j < N && i >= j) {
    if (j < n_d) {
      if (i < n_d) {
        v = ld_d(a.H + s * a.s_H + i + j * a.ldh, pol_stream);
        if (i == j) v = __dadd_rn(__dadd_rn(v, a.sigma_d[s * a.s_sd + j]), dw);
      } else {
        v = ld_d(a.Jd + s * a.s_J + (i - n_d) + j * a.ldj, pol_stream);
      }
    } else if (i == j) {
      const int64_t cy = j - n_d;
      v = -dc;
      if (cy >= a.m_E) {
        const double dh = a.d_h[s * a.s_dh + cy - a.m_E];
        if (!(dh > 0.0)) mds_set_status(a.status + s * a.s_st, MDS_ERR_NONPOSITIVE);
        v = __dsub_rn(v, 1.0 / dh);
      }
      v = __dsub_rn(v, a.dsum[s * a.m + cy]);
    }
  }
  return v;
}

// ---------------------------------------------------------------------------
// The tile kernel (see the top of the file).  Persistent CTAs take work items
// from a queue: for batched calls item g -> (tile order position g / batch,
// scenario g % batch); for a single system item g = items[g] (a tile, or one
// part of a split tile).  T is the tile in shared memory, column-major.
template <bool NORM>
__global__ void __launch_bounds__(CW * 32, 4) k_condense_tiles(CondArgs a) {
  pdl_wait();
  pdl_trigger();
  __shared__ double T[CT * CT];
  __shared__ double stcarry[CW];
  __shared__ int stckey[CW];
  __shared__ double red[CW][CT];
  __shared__ unsigned s_item;
  __shared__ bool s_last;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned long long pol_keep = pol_evict_last(), pol_stream = pol_evict_first();
  const int64_t nitem = a.split ? a.nitems : a.ntile * a.batch;
  for (;;) {
    if (threadIdx.x == 0) s_item = atomicAdd(&a.queue[0], 1u);
    __syncthreads();
    const int64_t g = s_item;
    if (g >= nitem) break;
    int64_t s = 0;
    uint32_t ij, part = 0, nparts = 1;
    if (a.split) {
      const uint2 it = a.items[g];
      ij = it.x; part = it.y >> 16; nparts = it.y & 0xffff;
    } else {
      s = g % a.batch;
      ij = a.order[g / a.batch];
      if (a.active && !a.active[s]) continue;   // (uniform across the CTA)
    }
    const int64_t I = ij >> 16, J = ij & 0xffff;
    const int64_t tile = anorm::tile_id(I, J);
    const int64_t i0 = I * CT, j0 = J * CT;
    const int64_t n_d = a.n_d, N = a.N;
    const double dw = a.dw_arr ? a.dw_arr[s] : a.delta_w;
    const double dc = a.dc_arr ? a.dc_arr[s] : a.delta_c;
    // ---- initial values: dense blocks of Eq.(6), or the M_yy diagonal start
    //      (-delta_c - 1/d_h - the diagonal pairs); a part of a split tile starts at 0
#pragma unroll
    for (int u = 0; u < 8; u++) {
      const int c = warp + 8 * u;
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int rr = lane + 32 * h;
        T[c * CT + rr] = nparts == 1 ? init_value(a, s, i0 + rr, j0 + c, dw, dc, pol_stream) : 0.0;
      }
    }
    __syncthreads();
    // ---- M_yy off-diagonal pairs: this item's range of the tile's sorted list, cut
    //      into CW contiguous runs of whole 64-pair double chunks (one per warp)
    uint32_t E0 = a.toff[tile], E1 = a.toff[tile + 1];
    if (nparts > 1) {
      const uint32_t nch = (E1 - E0 + 63u) / 64u, per = (nch + nparts - 1u) / nparts;
      const uint32_t q0 = E0 + 64u * min(nch, per * part);
      E1 = min(E1, E0 + 64u * min(nch, per * (part + 1)));
      E0 = q0;
    }
    if (E1 > E0) {
      const uint32_t nch = (E1 - E0 + 63u) / 64u, per = (nch + CW - 1u) / CW;
      const uint32_t r0 = E0 + 64u * min(nch, per * (uint32_t)warp);
      const uint32_t r1 = min(E1, E0 + 64u * min(nch, per * (uint32_t)(warp + 1)));
      const int ckey = (r0 > E0 && r0 < r1) ? (int)(ld_pair(a.pairs + r0 - 1, pol_stream) >> 52) : -1;
      int carried;
      const double carry = pair_range(a.pairs, r0, r1, ckey, a.Q + s * a.nnz, T, lane,
                                      pol_stream, pol_keep, &carried);
      if (lane == 0) { stcarry[warp] = carry; stckey[warp] = carried; }
      __syncthreads();
      if (threadIdx.x == 0) {   // carries in warp order (the previous warps' commits are done)
        for (int w = 1; w < CW; w++)
          if (stckey[w] >= 0) T[(stckey[w] >> 6) * CT + (stckey[w] & 63)] -= stcarry[w];
      }
    }
    __syncthreads();
    if (nparts > 1) {
      // part of a split tile: publish its sums; the last part merges them in part order
      double* pb = a.pbuf + (size_t)(a.pbase[tile] + part) * (CT * CT);
      for (int e = threadIdx.x; e < CT * CT; e += CW * 32) pb[e] = T[e];
      __threadfence();
      __syncthreads();
      if (threadIdx.x == 0) s_last = atomicAdd(&a.ticket[tile], 1u) == nparts - 1;
      __syncthreads();
      if (!s_last) continue;
      __threadfence();
      const double* pb0 = a.pbuf + (size_t)a.pbase[tile] * (CT * CT);
      for (int e = threadIdx.x; e < CT * CT; e += CW * 32) {
        double v = init_value(a, s, i0 + e % CT, j0 + e / CT, dw, dc, pol_stream);
        for (uint32_t q = 0; q < nparts; q++) v += __ldcg(pb0 + (size_t)q * (CT * CT) + e);
        T[e] = v;
      }
      __syncthreads();
    }
    // ---- epilogue: one coalesced store of the tile (lower part), and the norm
    //      partials of anorm::tile_partials (same sums, same order) formed on the fly
    double* M = a.M + s * a.s_M;
    anorm::Parts P = parts_of(a, s);
    bool bad = false;
    double ra0 = 0.0, ra1 = 0.0;
#pragma unroll
    for (int u = 0; u < 8; u++) {
      const int c = warp + 8 * u;
      const int64_t j = j0 + c;
      double ax[2];
      bool st[2];
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int rr = lane + 32 * h;
        const int64_t i = i0 + rr;
        const bool in = i < N && j < N && i >= j;
        const double x = T[c * CT + rr];
        ax[h] = in ? fabs(x) : 0.0;
        st[h] = in && i > j;
        if (in) {
          st_stream(M + i + j * a.ldm, x);
          if (!isfinite(x)) bad = true;
        }
      }
      if (NORM) {
        ra0 += ax[0];
        ra1 += ax[1];
        double cs = (st[0] ? ax[0] : 0.0) + (st[1] ? ax[1] : 0.0);
        cs = warp_sum(cs);
        if (lane == 0) P.pcol[tile * CT + c] = cs;
      }
    }
    if (NORM) {
      if (bad) atomicOr(&P.ctr[2], 1u);
      red[warp][lane] = ra0;
      red[warp][lane + 32] = ra1;
      __syncthreads();
      if (threadIdx.x < CT) {
        double sum = 0.0;
#pragma unroll
        for (int w = 0; w < CW; w++) sum += red[w][threadIdx.x];
        P.prow[tile * CT + threadIdx.x] = sum;
      }
    }
    __syncthreads();
  }
}
}  // namespace

// workspace: [queue 256 B | Q (16 nnz per scenario) | dsum (8 m per scenario) |
//             tickets (4 ntile) | part buffers (32 KB each) | norm parts per scenario]
static size_t al256(size_t x) { return (x + 255) / 256 * 256; }
struct CondLayout {
  size_t q, dsum, ticket, pbuf, parts, total;
};
static CondLayout cond_layout(const mds_plan* P, int64_t batch) {
  const int64_t m = P->m_E + P->m_I, N = std::max<int64_t>(P->n_d + m, 1);
  CondLayout L;
  L.q = 256;
  L.dsum = L.q + al256((size_t)batch * P->nnz * 16);
  L.ticket = L.dsum + al256((size_t)batch * std::max<int64_t>(m, 1) * 8);
  L.pbuf = L.ticket + al256((size_t)P->ntile * 4);
  L.parts = L.pbuf + (batch == 1 ? (size_t)P->nbuf * CT * CT * 8 : 0);
  L.total = L.parts + (size_t)batch * anorm::parts_bytes(N);
  return L;
}

extern "C" size_t mds_condense_workspace_size(const mds_plan* P, int64_t batch) {
  if (!P || batch < 1) return 0;
  return cond_layout(P, batch).total;
}

static int condense_launch(const mds_plan* P, CondArgs& a, void* work, size_t work_bytes, cudaStream_t st) {
  const int64_t n_s = P->n_s, n_d = P->n_d, m = P->m_E + P->m_I, N = n_d + m;
  a.n_s = n_s; a.n_d = n_d; a.m_E = P->m_E; a.m = m; a.N = N; a.nnz = P->nnz; a.ntile = P->ntile;
  a.nitems = P->nitems;
  a.rowptr = P->rowptr; a.tptr = P->tptr; a.tkp = P->tkp; a.pairs = P->pairs; a.toff = P->toff;
  a.pbase = P->pbase; a.order = P->order; a.items = P->items;
  a.split = a.batch == 1 ? 1 : 0;
  if (N == 0) return MDS_OK;
  if (!a.M || a.ldm < N) return MDS_ERR_ARG;
  if (n_s > 0 && (!a.h_ss || !a.sigma_s || !a.w || (P->nnz > 0 && !a.val))) return MDS_ERR_ARG;
  if (n_d > 0 && (!a.H || a.ldh < n_d || !a.sigma_d)) return MDS_ERR_ARG;
  if (n_d > 0 && m > 0 && (!a.Jd || a.ldj < m)) return MDS_ERR_ARG;
  if (P->m_I > 0 && !a.d_h) return MDS_ERR_ARG;
  if (!work || work_bytes < mds_condense_workspace_size(P, a.batch)) return MDS_ERR_WORKSPACE;
  if (a.rhs && !a.r) a.rhs = nullptr;
  const CondLayout L = cond_layout(P, a.batch);
  char* base = reinterpret_cast<char*>(work);
  a.queue = reinterpret_cast<unsigned*>(base);
  a.Q = reinterpret_cast<double2*>(base + L.q);
  a.dsum = reinterpret_cast<double*>(base + L.dsum);
  a.ticket = reinterpret_cast<unsigned*>(base + L.ticket);
  a.pbuf = reinterpret_cast<double*>(base + L.pbuf);
  a.parts = base + L.parts;
  a.parts_stride = anorm::parts_bytes(std::max<int64_t>(N, 1));
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  {
    const int64_t warps = std::max<int64_t>(a.batch * mds_cdiv(n_s, 32), 1);
    const int64_t blocks = std::max<int64_t>(std::max<int64_t>(mds_cdiv(warps, 8), mds_cdiv(a.ntile, 256)),
                                             mds_cdiv(a.batch * 4, 256));
    MDS_LAUNCH(PC_CONDENSE_W, st, MDS_CUDA_TRY(launch_pdl(k_condense_rows, dim3((unsigned)std::min<int64_t>(blocks, (int64_t)sms * 16)),
                                                          dim3(256), 0, st, a)));
  }
  {
    const int64_t bx = std::max<int64_t>(mds_cdiv(std::max<int64_t>(m, 1), 8), 1);
    MDS_LAUNCH(PC_CONDENSE_DIAG, st,
               MDS_CUDA_TRY(launch_pdl(k_condense_diag, dim3((unsigned)bx, (unsigned)a.batch), dim3(256), 0, st, a)));
  }
  int occ = 1;
  const bool norm = a.anorm != nullptr;
  if (norm) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_condense_tiles<true>, CW * 32, 0);
  else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_condense_tiles<false>, CW * 32, 0);
  const int64_t items = a.split ? P->nitems : P->ntile * a.batch;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(items, (int64_t)sms * std::max(occ, 1)));
  if (norm)
    MDS_LAUNCH(PC_CONDENSE_YY, st, MDS_CUDA_TRY(launch_pdl(k_condense_tiles<true>, dim3(grid), dim3(CW * 32), 0, st, a)));
  else
    MDS_LAUNCH(PC_CONDENSE_YY, st, MDS_CUDA_TRY(launch_pdl(k_condense_tiles<false>, dim3(grid), dim3(CW * 32), 0, st, a)));
  if (norm) {
    anorm::NormOut o = {};
    o.anorm = a.anorm;
    o.active = a.active;
    MDS_LAUNCH(PC_CONDENSE_DENSE, st, MDS_CUDA_TRY(anorm::launch_rows(N, a.parts, a.parts_stride, o, a.batch, st)));
  }
  return MDS_OK;
}
extern "C" int mds_condense(const mds_plan* P, const double* js_val, const double* h_ss, const double* sigma_s,
                            const double* H_dd, int64_t ldh, const double* sigma_d, const double* J_d, int64_t ldj,
                            const double* d_h, double delta_w, double delta_c, const double* r,
                            double* M, int64_t ldm, double* rhs_c, double* w_out, double* anorm_out,
                            int32_t* status, void* work, size_t work_bytes, void* stream) {
  if (!P) return MDS_ERR_ARG;
  CondArgs a = {};
  a.batch = 1;
  a.val = js_val; a.h_ss = h_ss; a.sigma_s = sigma_s; a.H = H_dd; a.ldh = ldh; a.sigma_d = sigma_d;
  a.Jd = J_d; a.ldj = ldj; a.d_h = d_h; a.delta_w = delta_w; a.delta_c = delta_c; a.r = r;
  a.M = M; a.ldm = ldm; a.rhs = rhs_c; a.w = w_out; a.anorm = anorm_out; a.status = status;
  return condense_launch(P, a, work, work_bytes, (cudaStream_t)stream);
}

extern "C" int mds_condense_batched(const mds_plan* P, int64_t batch,
                                    const double* js_val, int64_t str_val,
                                    const double* h_ss, int64_t str_hss, const double* sigma_s, int64_t str_sig,
                                    const double* H_dd, int64_t ldh, int64_t str_H,
                                    const double* sigma_d, int64_t str_sd,
                                    const double* J_d, int64_t ldj, int64_t str_J,
                                    const double* d_h, int64_t str_dh,
                                    const double* delta_w, const double* delta_c,
                                    const double* r, int64_t str_r,
                                    double* M, int64_t ldm, int64_t str_M,
                                    double* rhs_c, int64_t str_rhs, double* w_out, int64_t str_w,
                                    double* anorm_out, int32_t* status, const int32_t* active,
                                    void* work, size_t work_bytes, void* stream) {
  if (!P || batch < 0) return MDS_ERR_ARG;
  if (batch == 0) return MDS_OK;
  if (!status) return MDS_ERR_ARG;
  CondArgs a = {};
  a.batch = batch;
  a.val = js_val; a.s_val = str_val; a.h_ss = h_ss; a.s_hss = str_hss; a.sigma_s = sigma_s; a.s_sig = str_sig;
  a.H = H_dd; a.ldh = ldh; a.s_H = str_H; a.sigma_d = sigma_d; a.s_sd = str_sd;
  a.Jd = J_d; a.ldj = ldj; a.s_J = str_J; a.d_h = d_h; a.s_dh = str_dh;
  a.dw_arr = delta_w; a.dc_arr = delta_c; a.r = r; a.s_r = str_r;
  a.M = M; a.ldm = ldm; a.s_M = str_M; a.rhs = rhs_c; a.s_rhs = str_rhs; a.w = w_out; a.s_w = str_w;
  a.anorm = anorm_out; a.status = status; a.s_st = 1; a.active = active;
  return condense_launch(P, a, work, work_bytes, (cudaStream_t)stream);
}
