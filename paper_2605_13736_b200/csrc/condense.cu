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
//     row in the tile -- and, for one destination, by k (stable), which is
//     exactly the order in which the elimination of Eq.(5) visits them
//     (one sparse variable at a time);
//   * one 64-bit word per pair: p | (p - p') << 32 | row << 52 | col << 58.
// Per call (device, stream-ordered, two kernels + one for the norm):
//   k_condense_rows   one pass over the sparse variables (a1): q_k, w_k = 1/q_k,
//                     status on q_k <= 0, and per CSR entry Q[p] = (val_p w_k,
//                     val_p) and rho[p] = val_p (w_k r_xs[k]) (the rhs term).
//   k_condense_tiles  persistent CTAs take 64x64 tiles of lower M from a queue
//                     (heaviest first): the dense blocks are copied
//                     (H_dd + diag(sigma_d) + delta_w I, J_d), the M_yy tiles are
//                     initialised (-delta_c, -1/d_h) and then walk their sorted
//                     pair list: a warp reads 32 pair words (coalesced), gathers
//                     the two Q values, forms the products and each run of equal
//                     destination is subtracted IN K ORDER by its head lane from
//                     the shared-memory tile -- so every element of M (and of
//                     rhs_c) is computed with exactly the operations, in exactly
//                     the order, of the plain elimination (bit-identical to it).
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
  int64_t npairs, ntile;
  unsigned long long* pairs;   // [npairs]
  uint32_t* col_off;           // [ntile_with_pairs * 65] absolute pair offsets per tile column
  uint32_t* tile_cb;           // [ntile] index of the tile's 65-entry col_off block, or NONE
  uint32_t* order;             // [ntile] (I << 16 | J), heaviest tiles first
};

namespace {
constexpr int CT = anorm::AT;         // tile edge (64)
constexpr int CW = anorm::AW;         // warps per CTA (8)
constexpr uint32_t TILE_NONE = 0xffffffffu;
constexpr int PAIR_SBITS = 20;        // p - p' < 2^20 (row length limit of the pair encoding)
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

  // ---- condensation pair lists: counting sort by tile, then by (column, row) inside a tile
  const int64_t nb = (N + CT - 1) / CT, ntile = anorm::ntiles(N);
  auto tile_of = [&](int64_t row, int64_t col) { return anorm::tile_id(row / CT, col / CT); };
  std::vector<int64_t> tcount(ntile + 1, 0);
  int64_t npairs = 0;
  for (int64_t k = 0; k < n_s; k++)
    for (int64_t p = rowptr[k]; p < rowptr[k + 1]; p++)
      for (int64_t pp = rowptr[k]; pp <= p; pp++) {
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
        for (int64_t pp = rowptr[k]; pp <= p; pp++) {
          const int64_t row = n_d + colidx[p], col = n_d + colidx[pp];
          const unsigned long long w = (unsigned long long)(uint32_t)p |
                                       ((unsigned long long)(p - pp) << 32) |
                                       ((unsigned long long)(row % CT) << 52) |
                                       ((unsigned long long)(col % CT) << 58);
          pairs[fill[tile_of(row, col)]++] = w;
        }
  }
  std::vector<uint32_t> tile_cb(ntile, TILE_NONE), col_off;
  {
    std::vector<unsigned long long> tmp;
    for (int64_t t = 0; t < ntile; t++) {
      const int64_t a = tcount[t], b = tcount[t + 1];
      if (a == b) continue;
      // stable counting sort of this tile's pairs by (col, row) = bits 52..63
      int64_t cnt[CT * CT + 1];
      std::fill(cnt, cnt + CT * CT + 1, 0);
      auto key = [](unsigned long long w) { return (int)(((w >> 58) & 63) * CT + ((w >> 52) & 63)); };
      for (int64_t q = a; q < b; q++) cnt[key(pairs[q]) + 1]++;
      for (int i = 0; i < CT * CT; i++) cnt[i + 1] += cnt[i];
      tmp.assign(b - a, 0ull);
      std::vector<int64_t> pos(cnt, cnt + CT * CT);
      for (int64_t q = a; q < b; q++) tmp[pos[key(pairs[q])]++] = pairs[q];
      std::copy(tmp.begin(), tmp.end(), pairs.begin() + a);
      tile_cb[t] = (uint32_t)col_off.size();
      for (int c = 0; c <= CT; c++) col_off.push_back((uint32_t)(a + cnt[c * CT]));
    }
  }
  // processing order: heaviest tiles first (pairs, plus a per-element cost for the copy/store)
  std::vector<uint32_t> order;
  {
    std::vector<std::pair<int64_t, uint32_t>> cost;
    cost.reserve(ntile);
    for (int64_t I = 0; I < nb; I++)
      for (int64_t J = 0; J <= I; J++) {
        const int64_t t = anorm::tile_id(I, J);
        cost.emplace_back(-(4 * (tcount[t + 1] - tcount[t]) + CT * CT / 8), (uint32_t)((I << 16) | J));
      }
    std::stable_sort(cost.begin(), cost.end(),
                     [](const std::pair<int64_t, uint32_t>& x, const std::pair<int64_t, uint32_t>& y) {
                       return x.first < y.first;
                     });
    for (auto& c : cost) order.push_back(c.second);
  }

  mds_plan* P = new (std::nothrow) mds_plan();
  if (!P) return MDS_ERR_ARG;
  P->n_s = n_s; P->n_d = n_d; P->m_E = m_E; P->m_I = m_I; P->nnz = nnz; P->max_col_len = maxlen;
  P->npairs = npairs; P->ntile = ntile;
  P->rowptr = nullptr; P->colidx = nullptr; P->tptr = nullptr; P->tkp = nullptr;
  P->pairs = nullptr; P->col_off = nullptr; P->tile_cb = nullptr; P->order = nullptr;
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
            up((void**)&P->col_off, col_off.data(), sizeof(uint32_t) * col_off.size()) &&
            up((void**)&P->tile_cb, tile_cb.data(), sizeof(uint32_t) * ntile) &&
            up((void**)&P->order, order.data(), sizeof(uint32_t) * order.size());
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
  cudaFree(P->pairs); cudaFree(P->col_off); cudaFree(P->tile_cb); cudaFree(P->order);
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
  int64_t n_s, n_d, m_E, m, N, nnz, ntile, batch;
  const int32_t* rowptr;
  const unsigned long long* pairs;
  const uint32_t* col_off;
  const uint32_t* tile_cb;
  const uint32_t* order;
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
  double2* Q;        // [batch][nnz]
  double* rho;       // [batch][nnz]
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
__device__ __forceinline__ double2 ld_q(const double2* a, unsigned long long pol) {
  double2 v;
  asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(a), "l"(pol));
  return v;
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

// ---------------------------------------------------------------------------
// a1 + per-entry products: one thread per sparse variable (grid-stride over
// batch * n_s).  Same operations as the elimination: q = (h_ss + sigma_s) +
// delta_w, w = 1/q (IEEE division), t = val w, rhs term val (w r_xs).
// Also zeroes the tile queue and every scenario's norm counters.
__global__ void k_condense_rows(CondArgs a) {
  pdl_wait();
  pdl_trigger();
  const int64_t gt = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (gt < 4) a.queue[gt] = 0u;
  if (a.anorm && gt < a.batch * 4) {
    anorm::Parts P = parts_of(a, gt / 4);
    P.ctr[gt % 4] = 0u;
  }
  const int64_t total = a.batch * a.n_s;
  for (int64_t g = gt; g < total; g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = g / a.n_s, k = g - s * a.n_s;
    const double dw = a.dw_arr ? a.dw_arr[s] : a.delta_w;
    const double q = __dadd_rn(__dadd_rn(a.h_ss[s * a.s_hss + k], a.sigma_s[s * a.s_sig + k]), dw);
    if (!(q > 0.0)) mds_set_status(a.status + s * a.s_st, MDS_ERR_NONPOSITIVE);
    const double wk = 1.0 / q;
    a.w[s * a.s_w + k] = wk;
    const double wr = a.r ? __dmul_rn(wk, a.r[s * a.s_r + k]) : 0.0;
    const double* val = a.val + s * a.s_val;
    double2* Q = a.Q + s * a.nnz;
    double* rho = a.rho + s * a.nnz;
    const int32_t p1 = a.rowptr[k + 1];
    for (int32_t p = a.rowptr[k]; p < p1; p++) {
      const double v = val[p];
      Q[p] = make_double2(__dmul_rn(v, wk), v);
      if (a.r) rho[p] = __dmul_rn(v, wr);
    }
  }
}

// ---------------------------------------------------------------------------
// The tile kernel (see the top of the file).  Queue item g -> (tile order
// position g / batch, scenario g % batch): the heaviest tiles of every
// scenario go first.  T is the tile in shared memory, column-major.
template <bool NORM>
__global__ void __launch_bounds__(CW * 32) k_condense_tiles(CondArgs a) {
  pdl_wait();
  pdl_trigger();
  __shared__ double T[CT * CT];
  __shared__ double stp[CW][32], sth[CW][32];
  __shared__ int stk[CW][32];
  __shared__ double racc[CT];
  __shared__ double red[CW][CT];
  __shared__ unsigned s_item;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned long long pol_keep = pol_evict_last(), pol_stream = pol_evict_first();
  const int64_t nitem = a.ntile * a.batch;
  for (;;) {
    if (threadIdx.x == 0) s_item = atomicAdd(&a.queue[0], 1u);
    __syncthreads();
    const int64_t g = s_item;
    if (g >= nitem) break;
    const int64_t s = g % a.batch;
    const uint32_t ij = a.order[g / a.batch];
    const int64_t I = ij >> 16, J = ij & 0xffff;
    const int64_t tile = anorm::tile_id(I, J);
    const int64_t i0 = I * CT, j0 = J * CT;
    const int64_t n_d = a.n_d, N = a.N;
    const bool diag = I == J;
    const double dw = a.dw_arr ? a.dw_arr[s] : a.delta_w;
    const double dc = a.dc_arr ? a.dc_arr[s] : a.delta_c;
    const double* r = a.r ? a.r + s * a.s_r + a.n_s : nullptr;   // (r_xd, r_yg, r_yh)
    double* rhs = (a.rhs && r) ? a.rhs + s * a.s_rhs : nullptr;
    // ---- initial values: dense blocks of Eq.(6), or the M_yy diagonal start
    const double* H = a.H + s * a.s_H;
    const double* Jd = a.Jd + s * a.s_J;
#pragma unroll
    for (int u = 0; u < 8; u++) {
      const int c = warp + 8 * u;
      const int64_t j = j0 + c;
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int rr = lane + 32 * h;
        const int64_t i = i0 + rr;
        double v = 0.0;
        if (i < N && j < N && i >= j) {
          if (j < n_d) {
            if (i < n_d) {
              v = ld_d(H + i + j * a.ldh, pol_stream);
              if (i == j) v = __dadd_rn(__dadd_rn(v, a.sigma_d[s * a.s_sd + j]), dw);
            } else {
              v = ld_d(Jd + (i - n_d) + j * a.ldj, pol_stream);
            }
          } else if (i == j) {
            const int64_t cy = j - n_d;
            v = -dc;
            if (cy >= a.m_E) {
              const double dh = a.d_h[s * a.s_dh + cy - a.m_E];
              if (!(dh > 0.0)) mds_set_status(a.status + s * a.s_st, MDS_ERR_NONPOSITIVE);
              v = __dsub_rn(v, 1.0 / dh);
            }
          }
        }
        T[c * CT + rr] = v;
      }
    }
    if (diag && rhs && threadIdx.x < CT) {
      const int64_t j = j0 + threadIdx.x;
      racc[threadIdx.x] = j < N ? r[j] : 0.0;
    }
    __syncthreads();
    // ---- M_yy: subtract the sorted pair products, each destination in k order
    const uint32_t cb = a.tile_cb[tile];
    if (cb != TILE_NONE) {
      const double2* Q = a.Q + s * a.nnz;
      const double* rho = a.rho + s * a.nnz;
      for (int u = 0; u < 8; u++) {
        const int c = warp + 8 * u;
        const uint32_t e0 = a.col_off[cb + c], e1 = a.col_off[cb + c + 1];
        const bool rdiag = diag && rhs != nullptr;
        for (uint32_t base = e0; base < e1; base += 32) {
          const uint32_t idx = base + lane;
          const bool valid = idx < e1;
          int key = -1;
          double prod = 0.0, rh = 0.0;
          if (valid) {
            const unsigned long long wd = ld_pair(a.pairs + idx, pol_stream);
            const uint32_t p = (uint32_t)wd;
            const uint32_t sft = (uint32_t)(wd >> 32) & ((1u << PAIR_SBITS) - 1u);
            key = (int)((wd >> 52) & 63);
            const double2 qa = ld_q(Q + p, pol_keep);
            const double vb = sft ? ld_q(Q + (p - sft), pol_keep).y : qa.y;
            prod = __dmul_rn(qa.x, vb);
            if (rdiag && key == c) rh = ld_d(rho + p, pol_keep);
          }
          stp[warp][lane] = prod;
          sth[warp][lane] = rh;
          stk[warp][lane] = key;
          const int prev = __shfl_up_sync(0xffffffffu, key, 1);
          const bool head = valid && (lane == 0 || prev != key);
          __syncwarp();
          if (head) {
            double acc = T[c * CT + key];
            const bool dg = rdiag && key == c;
            double ra = dg ? racc[c] : 0.0;
            for (int q = lane; q < 32 && stk[warp][q] == key; q++) {
              acc = __dsub_rn(acc, stp[warp][q]);
              if (dg) ra = __dsub_rn(ra, sth[warp][q]);
            }
            T[c * CT + key] = acc;
            if (dg) racc[c] = ra;
          }
          __syncwarp();
        }
      }
    }
    __syncthreads();
    // ---- epilogue: one coalesced store of the tile (lower part), norm partials
    double* M = a.M + s * a.s_M;
    double v[8][2];
    bool strict[8][2];
    bool bad = false;
#pragma unroll
    for (int u = 0; u < 8; u++) {
      const int c = warp + 8 * u;
      const int64_t j = j0 + c;
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int rr = lane + 32 * h;
        const int64_t i = i0 + rr;
        const bool in = i < N && j < N && i >= j;
        const double x = T[c * CT + rr];
        v[u][h] = in ? x : 0.0;
        strict[u][h] = in && i > j;
        if (in) {
          st_stream(M + i + j * a.ldm, x);
          if (!isfinite(x)) bad = true;
        }
      }
    }
    if (diag && rhs && threadIdx.x < CT) {
      const int64_t j = j0 + threadIdx.x;
      if (j < N) rhs[j] = racc[threadIdx.x];
    }
    if (NORM) {
      anorm::Parts P = parts_of(a, s);
      if (bad) atomicOr(&P.ctr[2], 1u);
      anorm::tile_partials(v, strict, tile, P, red);
    }
    __syncthreads();
  }
}
}  // namespace

// workspace: [queue 256 B | Q (16 nnz per scenario) | rho (8 nnz per scenario) | norm parts per scenario]
static size_t condense_qr_bytes(const mds_plan* P, int64_t batch) {
  return ((size_t)batch * P->nnz * 24 + 255) / 256 * 256;
}

extern "C" size_t mds_condense_workspace_size(const mds_plan* P, int64_t batch) {
  if (!P || batch < 1) return 0;
  const int64_t N = std::max<int64_t>(P->n_d + P->m_E + P->m_I, 1);
  return 256 + condense_qr_bytes(P, batch) + (size_t)batch * anorm::parts_bytes(N);
}

static int condense_launch(const mds_plan* P, CondArgs& a, void* work, size_t work_bytes, cudaStream_t st) {
  const int64_t n_s = P->n_s, n_d = P->n_d, m = P->m_E + P->m_I, N = n_d + m;
  a.n_s = n_s; a.n_d = n_d; a.m_E = P->m_E; a.m = m; a.N = N; a.nnz = P->nnz; a.ntile = P->ntile;
  a.rowptr = P->rowptr; a.pairs = P->pairs; a.col_off = P->col_off; a.tile_cb = P->tile_cb; a.order = P->order;
  if (N == 0) return MDS_OK;
  if (!a.M || a.ldm < N) return MDS_ERR_ARG;
  if (n_s > 0 && (!a.h_ss || !a.sigma_s || !a.w || (P->nnz > 0 && !a.val))) return MDS_ERR_ARG;
  if (n_d > 0 && (!a.H || a.ldh < n_d || !a.sigma_d)) return MDS_ERR_ARG;
  if (n_d > 0 && m > 0 && (!a.Jd || a.ldj < m)) return MDS_ERR_ARG;
  if (P->m_I > 0 && !a.d_h) return MDS_ERR_ARG;
  if (!work || work_bytes < mds_condense_workspace_size(P, a.batch)) return MDS_ERR_WORKSPACE;
  if (a.rhs && !a.r) a.rhs = nullptr;
  char* base = reinterpret_cast<char*>(work);
  a.queue = reinterpret_cast<unsigned*>(base);
  a.Q = reinterpret_cast<double2*>(base + 256);
  a.rho = reinterpret_cast<double*>(base + 256 + (size_t)a.batch * P->nnz * 16);
  a.parts = base + 256 + condense_qr_bytes(P, a.batch);
  a.parts_stride = anorm::parts_bytes(std::max<int64_t>(N, 1));
  {
    const int64_t rows = std::max<int64_t>(a.batch * n_s, a.batch * 4);
    const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(mds_cdiv(rows, 256), 148 * 16));
    MDS_LAUNCH(PC_CONDENSE_W, st, MDS_CUDA_TRY(launch_pdl(k_condense_rows, dim3((unsigned)blocks), dim3(256), 0, st, a)));
  }
  int dev = 0, sms = 148, occ = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const bool norm = a.anorm != nullptr;
  if (norm) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_condense_tiles<true>, CW * 32, 0);
  else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_condense_tiles<false>, CW * 32, 0);
  const int64_t items = P->ntile * a.batch;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(items, (int64_t)sms * std::max(occ, 1)));
  if (norm)
    MDS_LAUNCH(PC_CONDENSE_YY, st, MDS_CUDA_TRY(launch_pdl(k_condense_tiles<true>, dim3(grid), dim3(CW * 32), 0, st, a)));
  else
    MDS_LAUNCH(PC_CONDENSE_YY, st, MDS_CUDA_TRY(launch_pdl(k_condense_tiles<false>, dim3(grid), dim3(CW * 32), 0, st, a)));
  if (norm) {
    // one launch for every scenario: grid (row blocks, batch); a per-scenario ticket
    // picks the last CTA of each scenario
    anorm::NormOut o = {};
    o.anorm = a.anorm;
    MDS_LAUNCH(PC_CONDENSE_DENSE, st,
               MDS_CUDA_TRY(launch_pdl(anorm::k_anorm_rows, dim3((unsigned)mds_cdiv(N, 256), (unsigned)a.batch), dim3(256),
                                       0, st, N, a.parts, a.parts_stride, o)));
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
                                    double* anorm_out, int32_t* status,
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
  a.anorm = anorm_out; a.status = status; a.s_st = 1;
  return condense_launch(P, a, work, work_bytes, (cudaStream_t)stream);
}
