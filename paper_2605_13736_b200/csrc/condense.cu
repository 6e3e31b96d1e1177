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
// Per call (device, stream-ordered; the pure dense tiles on a side stream, see
// k_condense_dense, concurrently with this chain):
//   k_condense_rows   one pass over the sparse variables (a1): q_k, w_k = 1/q_k,
//                     status on q_k <= 0, and per CSR entry Q[p] = (val_p w_k,
//                     val_p).
//   k_condense_diag   one warp per constraint column: the diagonal pairs p = p'
//                     of M_yy(c, c) and the rhs term (J_s^T (w . r_xs))_c.
//   k_condense_tiles  persistent CTAs take 64x64 tiles of lower M from a queue
//                     (heaviest first; the tiles right of n_d): the M_yy tiles are
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

#include <cuda.h>

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
  int64_t npairs, ntile, nitems, norder, ndense;
  uint32_t nbuf;               // part buffers (64x64) of the split tiles
  unsigned long long* pairs;   // [npairs] off-diagonal pairs, by tile, then (column, row), then k
  uint32_t* toff;              // [ntile + 1] pair range of each tile
  uint32_t* pbase;             // [ntile] first part buffer of a split tile
  uint32_t* order;             // [norder] (I << 16 | J), heaviest tiles first (batched calls)
  uint2* items;                // [nitems] (I << 16 | J, part << 16 | nparts), heaviest first (single system)
  uint32_t* dorder;            // [ndense] (I << 16 | J): the pure dense tiles (64 J + 63 < n_d), column-block order
};

namespace {
constexpr int CT = anorm::AT;         // tile edge (64)
constexpr int CW = anorm::AW;         // warps per CTA (8)
constexpr int PAIR_SBITS = 20;        // p - p' < 2^20 (row length limit of the pair encoding)
constexpr int64_t PART = 16384;       // pairs per work item of a split tile (single-system calls)
constexpr int PAIR_U = 2;             // 32-pair chunks per pipeline stage of pair_range
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
  // The pure dense tiles (every column < n_d: copies of H_dd / J_d, no pairs) are
  // k_condense_dense's, in column-block order; the rest (M_yy and the block column
  // that straddles n_d) go through the pair kernel's queue.
  std::vector<uint32_t> order;                 // tiles: (I << 16 | J)
  std::vector<uint2> items;                    // parts: (I << 16 | J, part << 16 | nparts)
  std::vector<uint32_t> dorder;                // pure dense tiles
  std::vector<uint32_t> pbase(ntile, 0);
  uint32_t nbuf = 0;
  const int64_t JD = n_d / CT;
  for (int64_t J = 0; J < JD; J++)
    for (int64_t I = J; I < nb; I++) dorder.push_back((uint32_t)((I << 16) | J));
  {
    std::vector<std::pair<int64_t, uint32_t>> cost;
    std::vector<std::pair<int64_t, uint2>> icost;
    cost.reserve(ntile);
    for (int64_t I = 0; I < nb; I++)
      for (int64_t J = JD; J <= I; J++) {
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
  P->norder = (int64_t)order.size(); P->ndense = (int64_t)dorder.size(); P->dorder = nullptr;
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
            up((void**)&P->items, items.data(), sizeof(uint2) * items.size()) &&
            up((void**)&P->dorder, dorder.data(), sizeof(uint32_t) * dorder.size());
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
  cudaFree(P->dorder);
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
  int64_t n_s, n_d, m_E, m, N, nnz, ntile, nitems, norder, ndense, batch;
  const int32_t* active;                // [batch] or NULL: scenarios with active[s] == 0 are left untouched
  const int32_t* rowptr;
  const int32_t* tptr;
  const int2* tkp;
  const unsigned long long* pairs;
  const uint32_t* toff;
  const uint32_t* pbase;
  const uint32_t* order;
  const uint2* items;
  const uint32_t* dorder;
  int split;                            // 1: walk `items` (split tiles), 0: walk `order`
  int64_t group;                        // batched: scenarios per group (see k_condense_tiles)
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
  double2* Q;        // [batch][nnz]  (val_p w_k, val_p); batched: 4 scenarios interleaved per entry (qst)
  int qst;           // entry stride of one scenario's Q: 1, or 4 (batched: entry p of scenario s at
                     //   ((s / 4) nnz + p) 4 + s % 4, so the 4 scenarios of a tile group share sectors)
  double* dsum;      // [batch][m]    sum over column c of val^2 w (the diagonal pairs)
  double* pbuf;      // [nbuf][64*64] part sums of split tiles
  unsigned* ticket;  // [ntile]       parts finished per split tile
  char* parts;       // [batch][parts_bytes(N)]
  size_t parts_stride;
  unsigned* queue;   // [4] tile queue counter
  __device__ double* parts_prow(int64_t s) const { return anorm::parts_at(parts + (size_t)s * parts_stride, N).prow; }
  __device__ double* parts_pcol(int64_t s) const { return anorm::parts_at(parts + (size_t)s * parts_stride, N).pcol; }
};

// scenario s's view of Q (entry p at qbase(a, s)[p * a.qst])
constexpr int QI = 4;   // scenarios interleaved per Q entry (batched; 8 measured: tiles 4.2 -> 3.9 ms but the a1 pass 2.4 -> 2.6, step +0.4 ms)
__device__ __forceinline__ double2* qbase(const CondArgs& a, int64_t s) {
  return a.qst == 1 ? a.Q + s * a.nnz : a.Q + (size_t)(s / QI) * a.nnz * QI + (s % QI);
}
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
  if (a.qst == QI) {
    // batched (interleaved Q): a warp takes 32 sparse variables of the 4 scenarios of a group;
    // lane (entry e = lane / 4, scenario s0 + lane % 4) writes one 16-byte Q entry, so the
    // warp's 32 stores are 512 contiguous bytes.  Same arithmetic as below.
    const int64_t ngrp = (a.batch + QI - 1) / QI;
    for (int64_t g = gw; g < ngrp * nblk; g += nw) {
      const int64_t grp = g / nblk, k0 = (g - grp * nblk) * 32, s0 = grp * QI;
      const int64_t k = k0 + lane;
      const int nrow = (int)min((int64_t)32, a.n_s - k0);
      double wk[QI];
      int rp = 0;
#pragma unroll
      for (int u = 0; u < QI; u++) {
        const int64_t s = s0 + u;
        wk[u] = 0.0;
        if (lane < nrow && s < a.batch && !(a.active && !a.active[s])) {
          const double dw = a.dw_arr ? a.dw_arr[s] : a.delta_w;
          const double q = __dadd_rn(__dadd_rn(a.h_ss[s * a.s_hss + k], a.sigma_s[s * a.s_sig + k]), dw);
          if (!(q > 0.0)) mds_set_status(a.status + s * a.s_st, MDS_ERR_NONPOSITIVE);
          wk[u] = 1.0 / q;
          a.w[s * a.s_w + k] = wk[u];
        }
      }
      if (lane < nrow) rp = a.rowptr[k];
      const int p0 = __shfl_sync(0xffffffffu, rp, 0);
      const int p1 = a.rowptr[k0 + nrow];
      const int e = lane / QI, su = lane % QI;
      const int64_t s = s0 + su;
      const bool live_s = s < a.batch && !(a.active && !a.active[s]);
      const double* val = a.val + (live_s ? s : 0) * a.s_val;
      double2* Qg = a.Q + (size_t)grp * a.nnz * QI + su;
      for (int pb = p0; pb < p1; pb += 32 / QI) {
        const int p = pb + e;
        int lo = 0;
#pragma unroll
        for (int step = 16; step >= 1; step >>= 1) {
          const int cand = lo + step;
          const int rc = __shfl_sync(0xffffffffu, rp, cand < nrow ? cand : 0);
          if (cand < nrow && rc <= p) lo = cand;
        }
        double wr = 0.0;
#pragma unroll
        for (int u = 0; u < QI; u++) {
          const double x = __shfl_sync(0xffffffffu, wk[u], lo);
          if (su == u) wr = x;
        }
        if (p < p1 && live_s) {
          const double v = val[p];
          st_keep2(Qg + (size_t)p * QI, make_double2(__dmul_rn(v, wr), v), pol_keep);
        }
      }
    }
    return;
  }
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
    double2* Q = qbase(a, s);
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
        st_keep2(Q + (size_t)p * a.qst, make_double2(__dmul_rn(v, wr), v), pol_keep);
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
  const double2* Q = qbase(a, s);
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
        q[u] = ld_q(Q + (size_t)(kp[u].y & ((1 << 27) - 1)) * a.qst, pol_keep);
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
template <int U>
__device__ __forceinline__ double pair_range(const unsigned long long* __restrict__ pairs, uint32_t r0, uint32_t r1,
                                             int ckey, const double2* __restrict__ Q, double* T, int lane, unsigned long long pol_stream,
                                             unsigned long long pol_keep, int* carried, int qst) {
  // software pipeline: the pair words of the next U chunks are loaded while the
  // current chunks' operand gathers are in flight
  double carry = 0.0;
  *carried = -1;
  unsigned long long wd[U];
#pragma unroll
  for (int u = 0; u < U; u++) {
    const uint32_t idx = r0 + 32 * u + lane;
    wd[u] = idx < r1 ? ld_pair(pairs + idx, pol_stream) : 0ull;
  }
  for (uint32_t base = r0; base < r1; base += 32 * U) {
    double qa[U], qb[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      qa[u] = qb[u] = 0.0;
      if (base + 32 * u + lane < r1) {
        const uint32_t p = (uint32_t)wd[u];
        const uint32_t sft = (uint32_t)(wd[u] >> 32) & ((1u << PAIR_SBITS) - 1u);
        qa[u] = ld_d(&Q[(size_t)p * qst].x, pol_keep);
        qb[u] = ld_d(&Q[(size_t)(p - sft) * qst].y, pol_keep);
      }
    }
    int key[U];
#pragma unroll
    for (int u = 0; u < U; u++) key[u] = (base + 32 * u + lane < r1) ? (int)(wd[u] >> 52) : 4096 + lane;
    const uint32_t nb = base + 32 * U;
#pragma unroll
    for (int u = 0; u < U; u++) {
      const uint32_t idx = nb + 32 * u + lane;
      wd[u] = idx < r1 ? ld_pair(pairs + idx, pol_stream) : 0ull;
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
      if (base + 32 * u >= r1) break;
      double v = __dmul_rn(qa[u], qb[u]);
      const int k = key[u];
      // segmented inclusive scan over the runs of equal key (keys sorted): run heads
      // from one ballot, and only as many doubling steps as the longest run needs
      // (the same sums, in the same order, as the full 5-step scan)
      const int pk = __shfl_up_sync(0xffffffffu, k, 1);
      const unsigned heads = __ballot_sync(0xffffffffu, lane == 0 || pk != k);
      const int dist = lane - (31 - __clz(heads & (0xffffffffu >> (31 - lane))));
      const int maxd = __reduce_max_sync(0xffffffffu, (unsigned)dist);
      for (int d = 1; d <= maxd; d <<= 1) {
        const double o = __shfl_up_sync(0xffffffffu, v, d);
        if (dist >= d) v += o;
      }
      bool tail = (base + 32 * u + lane < r1) && (lane == 31 || ((heads >> (lane + 1)) & 1u));
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
// from a queue: for batched calls item g -> (scenario group, tile order position,
// scenario in the group); for a single system item g = items[g] (a tile, or one
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
  const int64_t nitem = a.split ? a.nitems : a.norder * a.batch;
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
      // (scenario group, tile in heaviest-first order, scenario in the group): the CTAs
      // in flight gather the Q operands of a few scenarios only, so those stay in L2
      const int64_t per = a.norder * a.group, grp = g / per, pos = g - grp * per;
      const int64_t gs = min(a.group, a.batch - grp * a.group);
      s = grp * a.group + pos % gs;
      ij = a.order[pos / gs];
      if (a.active && !a.active[s]) {   // (uniform across the CTA)
        __syncthreads();                // s_item is rewritten at the top of the loop
        continue;
      }
    }
    const int64_t I = ij >> 16, J = ij & 0xffff;
    const int64_t tile = anorm::tile_id(I, J);
    const int64_t i0 = I * CT, j0 = J * CT;
    const int64_t N = a.N;
    const double dw = a.dw_arr ? a.dw_arr[s] : a.delta_w;
    const double dc = a.dc_arr ? a.dc_arr[s] : a.delta_c;
    // ---- initial values: dense blocks of Eq.(6), or the M_yy diagonal start
    //      (-delta_c - 1/d_h - the diagonal pairs); a part of a split tile starts at 0
    // (a tile strictly below the diagonal, inside M and right of n_d: all zeros)
    const bool full = I > J && i0 + CT <= N;
    if (nparts > 1 || (full && j0 >= a.n_d)) {
      for (int e = threadIdx.x; e < CT * CT / 2; e += CW * 32) reinterpret_cast<double2*>(T)[e] = make_double2(0.0, 0.0);
    } else {
#pragma unroll
      for (int u = 0; u < 8; u++) {
        const int c = warp + 8 * u;
#pragma unroll
        for (int h = 0; h < 2; h++) {
          const int rr = lane + 32 * h;
          T[c * CT + rr] = init_value(a, s, i0 + rr, j0 + c, dw, dc, pol_stream);
        }
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
      const double carry = pair_range<PAIR_U>(a.pairs, r0, r1, ckey, qbase(a, s), T, lane,
                                              pol_stream, pol_keep, &carried, a.qst);
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
        const bool in = full || (i < N && j < N && i >= j);
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

// ---------------------------------------------------------------------------
// The pure dense tiles (all 64 columns < n_d): M_xx = H_dd + diag(sigma_d) +
// delta_w I and M_yx = J_d, streamed straight from the inputs to M (no shared
// tile), with the tile's norm partials.  It depends on no other condensation
// kernel, so condense_launch runs it on a side stream CONCURRENTLY with the
// rows -> diag -> pair-tile chain: that chain is gather-latency bound, this one
// bandwidth bound.  Persistent CTAs stride over (tile, scenario) items.
// Layout: warp w owns columns c = w + 8u (u = 0..7) of the tile; VEC: lane l
// rows 2l, 2l+1 (16-byte loads/stores; needs even n_d, m, ld's, strides and
// 16-byte aligned bases), else lane l rows l, l + 32.  All eight (sixteen)
// loads of a tile are issued before the first use.  Norm partials in a fixed
// order; a non-finite entry turns its partials into +Inf (k_anorm_rows then
// reports NaN = "not finite"), so no counter is shared with the other chain.
__device__ __forceinline__ double2 ld_d2(const double* a, unsigned long long pol) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
               : "=d"(v.x), "=d"(v.y) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ void st_stream2(double* a, double2 v) {
  asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};" ::"l"(a), "d"(v.x), "d"(v.y) : "memory");
}
__device__ __forceinline__ double inf_if_nan(double x) { return isnan(x) ? __longlong_as_double(0x7ff0000000000000ll) : x; }

template <bool VEC, bool NORM>
__global__ void __launch_bounds__(CW * 32) k_condense_dense(CondArgs a) {
  __shared__ double red[CW][CT];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned long long pol = pol_evict_first();
  const int64_t n_d = a.n_d, N = a.N;
  const int64_t nitem = a.ndense * a.batch;
  for (int64_t g = blockIdx.x; g < nitem; g += gridDim.x) {
    const int64_t s = g % a.batch;
    if (a.active && !a.active[s]) continue;                  // (uniform across the CTA)
    const uint32_t ij = a.dorder[g / a.batch];
    const int64_t I = ij >> 16, J = ij & 0xffff;
    const int64_t i0 = I * CT, j0 = J * CT, tile = anorm::tile_id(I, J);
    const double dw = a.dw_arr ? a.dw_arr[s] : a.delta_w;
    const double* H = a.H + s * a.s_H;
    const double* Jd = a.Jd + s * a.s_J;
    const double* sd = a.sigma_d + s * a.s_sd;
    double* M = a.M + s * a.s_M;
    constexpr int R = VEC ? 1 : 2;      // row slots per lane
    double2 v[8][R];
    // ---- all loads first (predicated; zero outside the lower triangle / matrix)
#pragma unroll
    for (int u = 0; u < 8; u++) {
      const int64_t j = j0 + warp + 8 * u;
#pragma unroll
      for (int h = 0; h < R; h++) {
        const int64_t i = VEC ? i0 + 2 * lane : i0 + lane + 32 * h;
        v[u][h] = make_double2(0.0, 0.0);
        if (VEC) {
          if (i + 1 >= j && i < N) {   // at least one of rows i, i+1 is on/below the diagonal (N even)
            const double* src = i < n_d ? H + i + j * a.ldh : Jd + (i - n_d) + j * a.ldj;
            v[u][h] = ld_d2(src, pol);
          }
        } else if (i >= j && i < N) {
          v[u][h].x = ld_d(i < n_d ? H + i + j * a.ldh : Jd + (i - n_d) + j * a.ldj, pol);
        }
      }
    }
    // ---- diagonal terms, stores, partials
    double ra[2] = {0.0, 0.0};
#pragma unroll
    for (int u = 0; u < 8; u++) {
      const int c = warp + 8 * u;
      const int64_t j = j0 + c;
      double cs = 0.0;
#pragma unroll
      for (int h = 0; h < R; h++) {
        if (VEC) {
          const int64_t i = i0 + 2 * lane;
          double2 x = v[u][h];
          if (i == j) x.x = __dadd_rn(__dadd_rn(x.x, sd[j]), dw);
          if (i + 1 == j) x.y = __dadd_rn(__dadd_rn(x.y, sd[j]), dw);
          if (i < N) {
            if (i >= j) {
              st_stream2(M + i + j * a.ldm, x);
            } else if (i + 1 == j) {
              st_stream(M + i + 1 + j * a.ldm, x.y);
              x.x = 0.0;
            } else {
              x = make_double2(0.0, 0.0);
            }
          }
          const double a0 = fabs(x.x), a1 = fabs(x.y);
          ra[0] += a0;
          ra[1] += a1;
          cs += (i > j ? a0 : 0.0) + (i + 1 > j ? a1 : 0.0);
        } else {
          const int64_t i = i0 + lane + 32 * h;
          double x = v[u][h].x;
          if (i == j) x = __dadd_rn(__dadd_rn(x, sd[j]), dw);
          if (i >= j && i < N) st_stream(M + i + j * a.ldm, x);
          const double ax = fabs(x);
          ra[h] += ax;
          cs += i > j ? ax : 0.0;
        }
      }
      if (NORM) {
        cs = warp_sum(cs);
        if (lane == 0) a.parts_pcol(s)[tile * CT + c] = inf_if_nan(cs);
      }
    }
    if (NORM) {
      if (VEC) {
        red[warp][2 * lane] = ra[0];
        red[warp][2 * lane + 1] = ra[1];
      } else {
        red[warp][lane] = ra[0];
        red[warp][lane + 32] = ra[1];
      }
      __syncthreads();
      if (threadIdx.x < CT) {
        double sum = 0.0;
#pragma unroll
        for (int w = 0; w < CW; w++) sum += red[w][threadIdx.x];
        a.parts_prow(s)[tile * CT + threadIdx.x] = inf_if_nan(sum);
      }
      __syncthreads();
    }
  }
}

// ---------------------------------------------------------------------------
// The same dense tiles through the Tensor Memory Accelerator (variant cdense_tma;
// needs n_d a multiple of 64 and every leading dimension / stride / base 16-byte
// aligned).  Measured slower than the register-staged kernel beside the pair
// chain (C3: 0.369 vs 0.317 ms per condensation): its 4 x 32 KB ring keeps fewer
// bytes in flight per SM than two register-staged CTAs, and the ring's shared
// memory crowds out the pair kernel's CTAs.  Kept as a measured alternative:
// one persistent CTA per SM, a ring of DS 32 KB stages.  Thread 0 keeps DS - 1
// tile loads in flight (cp.async.bulk.tensor, 64 x 64 box from H_dd or J_d,
// completion on the stage's mbarrier); an off-diagonal tile is stored back to M
// unchanged by one TMA store straight from the stage (bulk group per iteration),
// while the eight warps form its norm partials from shared memory.  The 64x64
// diagonal tiles of M_xx (diagonal terms, lower part only) are written by the
// warps.
constexpr int DS = 4;                       // stages
constexpr int DSTAGE = CT * CT * 8;         // bytes per stage (64 x 64 FP64)
constexpr int DSMEM = DS * DSTAGE + 1024;   // + alignment slack

__device__ __forceinline__ unsigned dsm_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void dmbar_wait(unsigned bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(bar), "r"(parity) : "memory");
}

template <bool NORM>
__global__ void __launch_bounds__(CW * 32, 1) k_condense_dense_tma(CondArgs a, const __grid_constant__ CUtensorMap mH,
                                                                   const __grid_constant__ CUtensorMap mJ,
                                                                   const __grid_constant__ CUtensorMap mM) {
  extern __shared__ unsigned char dsm_raw[];
  double* stg = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(dsm_raw) + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) unsigned long long full[DS];
  __shared__ double red[CW][CT];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t n_d = a.n_d, N = a.N, nitem = a.ndense * a.batch;
  const int64_t nmine = nitem > blockIdx.x ? (nitem - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  auto item = [&](int64_t it, int64_t& s, int64_t& I, int64_t& J) {
    const int64_t g = blockIdx.x + it * (int64_t)gridDim.x;
    s = g % a.batch;
    const uint32_t ij = a.dorder[g / a.batch];
    I = ij >> 16;
    J = ij & 0xffff;
  };
  auto issue = [&](int64_t it) {   // thread 0: load item `it` of this CTA into stage it % DS
    if (it >= nmine) return;
    int64_t s, I, J;
    item(it, s, I, J);
    const unsigned bar = dsm_u32(&full[it % DS]);
    const unsigned dst = dsm_u32(stg + (it % DS) * (CT * CT));
    if (a.active && !a.active[s]) {
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
      return;
    }
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(DSTAGE) : "memory");
    const bool x = I * CT < n_d;
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n"
        ::"r"(dst), "l"(x ? &mH : &mJ), "r"((int)(x ? I * CT : I * CT - n_d)), "r"((int)(J * CT)), "r"((int)s), "r"(bar)
        : "memory");
  };
  if (threadIdx.x == 0) {
    for (int q = 0; q < DS; q++)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(dsm_u32(&full[q])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    for (int q = 0; q < DS - 1; q++) issue(q);
  }
  __syncthreads();
  for (int64_t it = 0; it < nmine; it++) {
    const int st = (int)(it % DS);
    dmbar_wait(dsm_u32(&full[st]), (unsigned)((it / DS) & 1));
    int64_t s, I, J;
    item(it, s, I, J);
    const double* T = stg + st * (CT * CT);
    const bool act = !(a.active && !a.active[s]);
    const int64_t i0 = I * CT, j0 = J * CT, tile = anorm::tile_id(I, J);
    if (act && I != J && threadIdx.x == 0) {
      asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];\n"
                   ::"l"(&mM), "r"((int)i0), "r"((int)j0), "r"((int)s), "r"(dsm_u32(T)) : "memory");
    }
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
    if (act) {
      const double dw = a.dw_arr ? a.dw_arr[s] : a.delta_w;
      const double* sd = a.sigma_d + s * a.s_sd;
      double* M = a.M + s * a.s_M;
      double ra[2] = {0.0, 0.0};
#pragma unroll
      for (int u = 0; u < 8; u++) {
        const int c = warp + 8 * u;
        const int64_t j = j0 + c, i = i0 + 2 * lane;
        double2 x = *reinterpret_cast<const double2*>(T + c * CT + 2 * lane);
        double cs = 0.0;
        if (I == J) {   // diagonal tile of M_xx: diagonal terms, lower part only, stored here
          if (i == j) x.x = __dadd_rn(__dadd_rn(x.x, sd[j]), dw);
          if (i + 1 == j) x.y = __dadd_rn(__dadd_rn(x.y, sd[j]), dw);
          if (i >= j) {
            st_stream2(M + i + j * a.ldm, x);
          } else if (i + 1 == j) {
            st_stream(M + i + 1 + j * a.ldm, x.y);
            x.x = 0.0;
          } else {
            x = make_double2(0.0, 0.0);
          }
        } else if (i >= N) {
          x = make_double2(0.0, 0.0);   // (zero-filled rows below the matrix)
        }
        const double a0 = fabs(x.x), a1 = fabs(x.y);
        ra[0] += a0;
        ra[1] += a1;
        cs += (i > j ? a0 : 0.0) + (i + 1 > j ? a1 : 0.0);
        if (NORM) {
          cs = warp_sum(cs);
          if (lane == 0) a.parts_pcol(s)[tile * CT + c] = inf_if_nan(cs);
        }
      }
      if (NORM) {
        red[warp][2 * lane] = ra[0];
        red[warp][2 * lane + 1] = ra[1];
      }
    }
    __syncthreads();
    if (act && NORM && threadIdx.x < CT) {
      double sum = 0.0;
#pragma unroll
      for (int w = 0; w < CW; w++) sum += red[w][threadIdx.x];
      a.parts_prow(s)[tile * CT + threadIdx.x] = inf_if_nan(sum);
    }
    // refill the stage consumed in the previous iteration (its store has had one
    // iteration to read it) with the item DS - 1 ahead of this one
    if (threadIdx.x == 0) {
      asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");
      issue(it + DS - 1);
    }
    __syncthreads();   // red reused next iteration
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
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
  L.dsum = L.q + al256((size_t)(batch > 1 ? (batch + QI - 1) / QI * QI : 1) * P->nnz * 16);
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

// The side stream of the dense-tile kernel (one per host thread and device, so
// concurrent callers never share the fork/join events; graph-capturable: the
// fork is an event record + wait, the join likewise).
struct SideStream {
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
static SideStream* side_stream(int dev) {
  thread_local SideStream ss[64];
  if (dev < 0 || dev >= 64) return nullptr;
  SideStream& x = ss[dev];
  if (!x.s) {
    if (cudaStreamCreateWithFlags(&x.s, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&x.fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&x.join, cudaEventDisableTiming) != cudaSuccess) {
      x.s = nullptr;
      return nullptr;
    }
  }
  return &x;
}

typedef CUresult (*PFN_encTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static PFN_encTiled cond_encoder() {
  static const PFN_encTiled fn = []() -> PFN_encTiled {   // thread-safe one-time lookup
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    PFN_encTiled r = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      r = reinterpret_cast<PFN_encTiled>(p);
    (void)cudaGetLastError();
    return r;
  }();
  return fn;
}
// 3-D map over `batch` column-major (rows x cols, ld) FP64 matrices `bstride` elements
// apart (0: one matrix); 64 x 64 x 1 box, no swizzle, zero fill out of bounds
static bool cond_map(CUtensorMap* m, const double* base, int64_t rows, int64_t cols, int64_t ld, int64_t batch,
                     int64_t bstride) {
  PFN_encTiled enc = cond_encoder();
  if (!enc || rows < 1 || cols < 1) return false;
  cuuint64_t dims[3] = {(cuuint64_t)rows, (cuuint64_t)cols, (cuuint64_t)batch};
  cuuint64_t strides[2] = {(cuuint64_t)ld * 8, (cuuint64_t)(bstride > 0 ? bstride : ld * cols) * 8};
  cuuint32_t box[3] = {CT, CT, 1};
  cuuint32_t es[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static int condense_launch(const mds_plan* P, CondArgs& a, void* work, size_t work_bytes, cudaStream_t st) {
  const int64_t n_s = P->n_s, n_d = P->n_d, m = P->m_E + P->m_I, N = n_d + m;
  a.n_s = n_s; a.n_d = n_d; a.m_E = P->m_E; a.m = m; a.N = N; a.nnz = P->nnz; a.ntile = P->ntile;
  a.nitems = P->nitems;
  a.rowptr = P->rowptr; a.tptr = P->tptr; a.tkp = P->tkp; a.pairs = P->pairs; a.toff = P->toff;
  a.pbase = P->pbase; a.order = P->order; a.items = P->items; a.dorder = P->dorder;
  a.norder = P->norder; a.ndense = P->ndense;
  a.split = a.batch == 1 ? 1 : 0;
  a.qst = a.batch > 1 ? QI : 1;
  a.group = std::max<int64_t>(1, std::min<int64_t>(g_mds_var.cond_group, a.batch));
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
  const bool norm = a.anorm != nullptr;
  int prio_lo = INT_MIN, prio_hi = INT_MIN;   // (variant cond_prio)
  if (g_mds_var.cond_prio) cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
  // ---- fork: the pure dense tiles on the side stream, concurrent with the chain below
  SideStream* side = nullptr;
  if (a.ndense > 0) {
    side = side_stream(dev);
    if (!side) return MDS_ERR_CUDA;
    auto even = [](int64_t x) { return (x & 1) == 0; };
    auto al16 = [](const void* p) { return ((uintptr_t)p & 15) == 0; };
    const bool vec = even(n_d) && even(m) && even(a.ldh) && even(a.ldj) && even(a.ldm) && even(a.s_H) &&
                     even(a.s_J) && even(a.s_M) && al16(a.H) && al16(a.M) && (m == 0 || al16(a.Jd));
    const unsigned grid = (unsigned)std::max<int64_t>(
        1, g_mds_var.cdense_ctas == 0 ? a.ndense * a.batch   // (0: one CTA per tile, not persistent)
                                      : std::min<int64_t>(a.ndense * a.batch, (int64_t)sms * g_mds_var.cdense_ctas));
    cudaStream_t ds = st;
    if (!g_mds_var.cdense_serial) {
      MDS_CUDA_TRY(cudaEventRecord(side->fork, st));
      MDS_CUDA_TRY(cudaStreamWaitEvent(side->s, side->fork, 0));
      ds = side->s;
    } else {
      side = nullptr;
    }
    CUtensorMap mH, mJ, mM;
    const bool tma = vec && n_d % CT == 0 && g_mds_var.cdense_tma && cond_map(&mH, a.H, n_d, n_d, a.ldh, a.batch, a.s_H) &&
                     (m == 0 ? cond_map(&mJ, a.H, n_d, n_d, a.ldh, a.batch, a.s_H)
                             : cond_map(&mJ, a.Jd, m, n_d, a.ldj, a.batch, a.s_J)) &&
                     cond_map(&mM, a.M, N, N, a.ldm, a.batch, a.s_M);
    if (tma) {
      auto kt = norm ? k_condense_dense_tma<true> : k_condense_dense_tma<false>;
      if (mds_once_per_device((const void*)k_condense_dense_tma<true>)) {
        MDS_CUDA_TRY(cudaFuncSetAttribute(k_condense_dense_tma<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, DSMEM));
        MDS_CUDA_TRY(cudaFuncSetAttribute(k_condense_dense_tma<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, DSMEM));
      }
      const unsigned gt = (unsigned)std::max<int64_t>(1, std::min<int64_t>(a.ndense * a.batch, (int64_t)sms));
      MDS_LAUNCH(PC_CONDENSE_COPY, ds, (kt<<<gt, CW * 32, DSMEM, ds>>>(a, mH, mJ, mM)));
    } else {
      auto kd = vec ? (norm ? k_condense_dense<true, true> : k_condense_dense<true, false>)
                    : (norm ? k_condense_dense<false, true> : k_condense_dense<false, false>);
      if (prio_lo != INT_MIN)
        MDS_LAUNCH(PC_CONDENSE_COPY, ds, MDS_CUDA_TRY(launch_pdl_prio(kd, dim3(grid), dim3(CW * 32), 0, ds, prio_lo, a)));
      else
        MDS_LAUNCH(PC_CONDENSE_COPY, ds, (kd<<<grid, CW * 32, 0, ds>>>(a)));
    }
  }
  {
    const int64_t warps = std::max<int64_t>(a.batch * mds_cdiv(n_s, 32), 1);
    const int64_t blocks = std::max<int64_t>(std::max<int64_t>(mds_cdiv(warps, 8), mds_cdiv(a.ntile, 256)),
                                             mds_cdiv(a.batch * 4, 256));
    MDS_LAUNCH(PC_CONDENSE_W, st, MDS_CUDA_TRY(launch_pdl_prio(k_condense_rows, dim3((unsigned)std::min<int64_t>(blocks, (int64_t)sms * 16)),
                                                               dim3(256), 0, st, prio_hi, a)));
  }
  {
    const int64_t bx = std::max<int64_t>(mds_cdiv(std::max<int64_t>(m, 1), 8), 1);
    MDS_LAUNCH(PC_CONDENSE_DIAG, st,
               MDS_CUDA_TRY(launch_pdl_prio(k_condense_diag, dim3((unsigned)bx, (unsigned)a.batch), dim3(256), 0, st, prio_hi, a)));
  }
  int occ = 1;
  if (norm) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_condense_tiles<true>, CW * 32, 0);
  else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_condense_tiles<false>, CW * 32, 0);
  const int64_t items = a.split ? P->nitems : P->norder * a.batch;
  if (items > 0) {
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(items, (int64_t)sms * std::max(occ, 1)));
    if (norm)
      MDS_LAUNCH(PC_CONDENSE_YY, st, MDS_CUDA_TRY(launch_pdl_prio(k_condense_tiles<true>, dim3(grid), dim3(CW * 32), 0, st, prio_hi, a)));
    else
      MDS_LAUNCH(PC_CONDENSE_YY, st, MDS_CUDA_TRY(launch_pdl_prio(k_condense_tiles<false>, dim3(grid), dim3(CW * 32), 0, st, prio_hi, a)));
  }
  // ---- join
  if (side) {
    MDS_CUDA_TRY(cudaEventRecord(side->join, side->s));
    MDS_CUDA_TRY(cudaStreamWaitEvent(st, side->join, 0));
  }
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
