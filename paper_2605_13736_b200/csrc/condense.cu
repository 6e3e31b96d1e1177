// condense.cu — mds_plan_* and mds_condense: Eq.(5) -> Eq.(6) of PAPER.md
// (K3 "M := M + A D B^T", fused over CSR
// instead of the paper's three triplet launches).
//
// Kernels (HBM-bound; algorithmic bytes in DESIGN.md §Roofline):
//   k_condense_w      w_k = 1/(h_ss+sigma_s+delta_w), status on q<=0          (grid-stride)
//   k_condense_dense  columns j < n_d: M[j:n_d,j] = H_dd+diag, M[n_d:,j] = J_d,
//                     rhs_c[0:n_d] = r_xd                                     (CTA per column)
//   k_condense_yy     columns n_d+c: one WARP owns output column c of M_yy,
//                     accumulates -sum_k w_k J[k,c] J[k,c1] (c1 >= c) in a
//                     private shared-memory column (no FP64 smem atomics: lanes
//                     that collide on c1 are serialised via __match_any_sync),
//                     then writes the column once, coalesced; also rhs_c[n_d+c].
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <new>
#include <vector>

#include <cstdlib>

#include "common.cuh"

struct mds_plan {
  int64_t n_s, n_d, m_E, m_I, nnz;
  int32_t* rowptr;   // [n_s+1] device
  int32_t* colidx;   // [nnz]   device
  int32_t* tptr;     // [m+1]   constraint-major transpose: entries of column c
  int2* tkp;         // [nnz]   (k, p): sparse variable k, CSR position p of (k,c)
  int32_t max_col_len;
};

extern "C" const char* mds_version(void) { return "mds_b200 0.1 sm_100a"; }

extern "C" int mds_plan_create(int64_t n_s, int64_t n_d, int64_t m_E, int64_t m_I,
                               const int32_t* rowptr, const int32_t* colidx, mds_plan** out) {
  if (!out || n_s < 0 || n_d < 0 || m_E < 0 || m_I < 0) return MDS_ERR_ARG;
  if (n_s > 0 && (!rowptr)) return MDS_ERR_ARG;
  const int64_t m = m_E + m_I;
  if (m + n_d > (int64_t)1 << 30) return MDS_ERR_ARG;
  int64_t nnz = n_s > 0 ? rowptr[n_s] : 0;
  if (n_s > 0 && rowptr[0] != 0) return MDS_ERR_PATTERN;
  if (nnz > 0 && !colidx) return MDS_ERR_ARG;
  if (nnz >= ((int64_t)1 << 27)) return MDS_ERR_ARG;   // packed transpose map limit
  // validate canonical CSR (reading R13): sorted, unique, in range
  for (int64_t k = 0; k < n_s; k++) {
    if (rowptr[k + 1] < rowptr[k]) return MDS_ERR_PATTERN;
    for (int64_t p = rowptr[k]; p < rowptr[k + 1]; p++) {
      if (colidx[p] < 0 || colidx[p] >= m) return MDS_ERR_PATTERN;
      if (p > rowptr[k] && colidx[p] <= colidx[p - 1]) return MDS_ERR_PATTERN;
    }
  }
  // constraint-major transpose (counting sort; entries of a column in k order)
  std::vector<int32_t> tptr(m + 1, 0);
  for (int64_t p = 0; p < nnz; p++) tptr[colidx[p] + 1]++;
  for (int64_t c = 0; c < m; c++) tptr[c + 1] += tptr[c];
  std::vector<int2> tkp(std::max<int64_t>(nnz, 1));
  {
    std::vector<int32_t> fill(tptr.begin(), tptr.end() - 1);
    for (int64_t k = 0; k < n_s; k++)
      for (int64_t p = rowptr[k]; p < rowptr[k + 1]; p++) {
        // y = p | min(suffix length, 31) << 27  (31 = "look up rowptr")
        const unsigned sl = (unsigned)std::min<int64_t>(rowptr[k + 1] - p, 31);
        tkp[fill[colidx[p]]++] = make_int2((int)k, (int)((unsigned)p | (sl << 27)));
      }
  }
  int32_t maxlen = 0;
  for (int64_t c = 0; c < m; c++) maxlen = std::max(maxlen, tptr[c + 1] - tptr[c]);

  mds_plan* P = new (std::nothrow) mds_plan();
  if (!P) return MDS_ERR_ARG;
  P->n_s = n_s; P->n_d = n_d; P->m_E = m_E; P->m_I = m_I; P->nnz = nnz; P->max_col_len = maxlen;
  P->rowptr = nullptr; P->colidx = nullptr; P->tptr = nullptr; P->tkp = nullptr;
  bool ok = cudaMalloc(&P->rowptr, sizeof(int32_t) * (n_s + 1)) == cudaSuccess &&
            cudaMalloc(&P->colidx, sizeof(int32_t) * std::max<int64_t>(nnz, 1)) == cudaSuccess &&
            cudaMalloc(&P->tptr, sizeof(int32_t) * (m + 1)) == cudaSuccess &&
            cudaMalloc(&P->tkp, sizeof(int2) * std::max<int64_t>(nnz, 1)) == cudaSuccess;
  if (ok) {
    std::vector<int32_t> rp(n_s + 1, 0);
    if (n_s > 0) std::memcpy(rp.data(), rowptr, sizeof(int32_t) * (n_s + 1));
    ok = cudaMemcpy(P->rowptr, rp.data(), sizeof(int32_t) * (n_s + 1), cudaMemcpyHostToDevice) == cudaSuccess &&
         (nnz == 0 || cudaMemcpy(P->colidx, colidx, sizeof(int32_t) * nnz, cudaMemcpyHostToDevice) == cudaSuccess) &&
         cudaMemcpy(P->tptr, tptr.data(), sizeof(int32_t) * (m + 1), cudaMemcpyHostToDevice) == cudaSuccess &&
         (nnz == 0 || cudaMemcpy(P->tkp, tkp.data(), sizeof(int2) * nnz, cudaMemcpyHostToDevice) == cudaSuccess);
  }
  if (!ok) {
    cudaFree(P->rowptr); cudaFree(P->colidx); cudaFree(P->tptr); cudaFree(P->tkp);
    delete P;
    return MDS_ERR_CUDA;
  }
  *out = P;
  return MDS_OK;
}

extern "C" int mds_plan_destroy(mds_plan* P) {
  if (!P) return MDS_ERR_ARG;
  cudaFree(P->rowptr); cudaFree(P->colidx); cudaFree(P->tptr); cudaFree(P->tkp);
  delete P;
  return MDS_OK;
}

extern "C" int mds_plan_dims(const mds_plan* P, int64_t* out) {
  if (!P || !out) return MDS_ERR_ARG;
  out[0] = P->n_s; out[1] = P->n_d; out[2] = P->m_E; out[3] = P->m_I; out[4] = P->nnz;
  return MDS_OK;
}

// accessor for solve.cu (same library)
const int32_t* mds_plan_rowptr(const mds_plan* P) { return P->rowptr; }
const int32_t* mds_plan_colidx(const mds_plan* P) { return P->colidx; }
const int32_t* mds_plan_tptr(const mds_plan* P) { return P->tptr; }
const int2* mds_plan_tkp(const mds_plan* P) { return P->tkp; }

// ---------------------------------------------------------------------------
// w_k = 1/q_k, q_k = h_ss + sigma_s + delta_w  (Q_{x_s}^{-1}, A2 PAPER.md:121)
__global__ void k_condense_w(int64_t n_s, const double* __restrict__ h_ss, const double* __restrict__ sigma_s,
                             double delta_w, double* __restrict__ w, int32_t* status) {
  pdl_wait();
  pdl_trigger();
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n_s; k += (int64_t)gridDim.x * blockDim.x) {
    double q = h_ss[k] + sigma_s[k] + delta_w;
    if (!(q > 0.0)) mds_set_status(status, MDS_ERR_NONPOSITIVE);
    w[k] = 1.0 / q;
  }
}

// dense blocks of Eq.(6): column j < n_d of M (lower): rows j..n_d-1 from H_dd
// (+sigma_d+delta_w on the diagonal), rows n_d..N-1 from J_d column j.
__global__ void k_condense_dense(int64_t n_d, int64_t m, const double* __restrict__ H, int64_t ldh,
                                 const double* __restrict__ sigma_d, double delta_w,
                                 const double* __restrict__ Jd, int64_t ldj,
                                 double* __restrict__ M, int64_t ldm,
                                 const double* __restrict__ r_xd, double* __restrict__ rhs_c) {
  // Launched right after k_condense_yy (programmatic dependent launch) and independent of it
  // (inputs only; disjoint outputs), so it starts as soon as k_condense_yy has started -- whose
  // own griddepcontrol.wait already ordered everything before mds_condense -- and runs in the
  // SM slots the latency-bound k_condense_yy leaves free.  It waits for k_condense_yy only at
  // its end, so its completion (what the next kernel waits for) implies the whole condensation.
  pdl_trigger();
  for (int64_t j = blockIdx.x; j < n_d; j += gridDim.x) {
    double* Mj = M + j * ldm;
    const double* Hj = H + j * ldh;
    const double* Jj = Jd + j * ldj;
    for (int64_t i = j + threadIdx.x; i < n_d; i += blockDim.x) {
      double v = Hj[i];
      if (i == j) v = v + sigma_d[j] + delta_w;
      Mj[i] = v;
    }
    for (int64_t c = threadIdx.x; c < m; c += blockDim.x) Mj[n_d + c] = Jj[c];
    if (threadIdx.x == 0 && rhs_c) rhs_c[j] = r_xd[j];
  }
  pdl_wait();
}

// M_yy column c (rows c..m-1 of the (y,y) block).  One WARP owns output
// column c (and its fold partner m-1-c, so every warp does equal work) and
// accumulates -sum_k w_k J[k,c] J[k,c1] (c1 >= c) in a private shared-memory
// column; the column is then written once, coalesced.  Per iteration each lane
// takes U list entries (k, p, suffix length) of the constraint-major transpose
// and issues all their gathers at once (latency-bound on L2 otherwise).  The
// diagonal term (s = 0, every lane hits it) is a warp sum; off-diagonal lanes
// that collide on the same c1 are serialised via __match_any_sync (no FP64
// shared-memory atomics, which are CAS loops on sm_100a).  Deterministic.
// L2 cache policies: the J_s row gathers (colidx, val, w, r_xs: ~70 MB at C3)
// are re-read ~5x and must stay L2-resident while M (268 MB) streams out.
__device__ __forceinline__ unsigned long long pol_evict_last() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ double ldg_el(const double* a, unsigned long long pol) {
  double v;
  asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ int ldg_el(const int32_t* a, unsigned long long pol) {
  int v;
  asm volatile("ld.global.nc.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ void stg_ef(double* a, double v) {   // streaming store (evict-first)
  asm volatile("st.global.cs.f64 [%0], %1;" ::"l"(a), "d"(v) : "memory");
}

constexpr int YY_U = 2;      // list entries per lane per iteration
constexpr int YY_SMAX = 8;   // suffix entries gathered up front (longer suffixes take a slow loop)
constexpr unsigned TKP_PMASK = (1u << 27) - 1u;

template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 1)
k_condense_yy(int64_t n_d, int64_t m_E, int64_t m, int64_t acc_len,
              const int32_t* __restrict__ rowptr, const int32_t* __restrict__ colidx,
              const double* __restrict__ val, const int32_t* __restrict__ tptr, const int2* __restrict__ tkp,
              const double* __restrict__ w, const double* __restrict__ d_h, double delta_c,
              const double* __restrict__ r, int64_t n_s, double* __restrict__ M, int64_t ldm,
              double* __restrict__ rhs_c, int32_t* status) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ double smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* acc = smem + (size_t)warp * acc_len;
  const int64_t task = (int64_t)blockIdx.x * WARPS + warp;
  const int64_t ntask = (m + 1) / 2;
  if (task >= ntask) return;
  const unsigned lanemask_lt = (1u << lane) - 1u;
  const unsigned long long pol = pol_evict_last();
  for (int half = 0; half < 2; half++) {
    const int64_t c = half ? (m - 1 - task) : task;
    if (half && c == task) break;
    const int64_t len = m - c;
    double rsum = 0.0;
    const int32_t e0 = tptr[c], e1 = tptr[c + 1];
    for (int64_t base = 0; base < len; base += acc_len) {
      const int64_t clen = (len - base < acc_len) ? (len - base) : acc_len;
      for (int64_t i = lane; i < clen; i += 32) acc[i] = 0.0;
      __syncwarp();
      double diag = 0.0;
      // software pipeline over iterations: the transpose entries two iterations ahead
      // and the row gathers one iteration ahead are in flight while this iteration
      // scatters (the loop is otherwise bound by dependent L2/HBM latency)
      struct KP { int k[YY_U], p[YY_U], l[YY_U]; };
      struct GA { int cs[YY_U][YY_SMAX]; double vs[YY_U][YY_SMAX]; double wk[YY_U], rr[YY_U]; int l[YY_U]; };
      auto load_kp = [&](int32_t e, KP& o) {
#pragma unroll
        for (int u = 0; u < YY_U; u++) {
          const int32_t my = e + u * 32 + lane;
          o.l[u] = 0; o.k[u] = 0; o.p[u] = 0;
          if (my < e1) {
            const int2 kp = tkp[my];
            o.k[u] = kp.x;
            o.p[u] = (int)((unsigned)kp.y & TKP_PMASK);
            o.l[u] = (int)((unsigned)kp.y >> 27);
          }
        }
      };
      auto gather = [&](KP& kp, GA& g) {
#pragma unroll
        for (int u = 0; u < YY_U; u++) {
          if (kp.l[u] == 31) kp.l[u] = rowptr[kp.k[u] + 1] - kp.p[u];
          g.l[u] = kp.l[u];
#pragma unroll
          for (int s2 = 0; s2 < YY_SMAX; s2++) {
            g.cs[u][s2] = -1;
            g.vs[u][s2] = 0.0;
            if (s2 < kp.l[u]) {
              g.cs[u][s2] = ldg_el(colidx + kp.p[u] + s2, pol);
              g.vs[u][s2] = ldg_el(val + kp.p[u] + s2, pol);
            }
          }
          g.wk[u] = (kp.l[u] > 0) ? ldg_el(w + kp.k[u], pol) : 0.0;
          g.rr[u] = (base == 0 && r && kp.l[u] > 0) ? ldg_el(r + kp.k[u], pol) : 0.0;
        }
      };
      KP kpn, kpnn;
      GA ga, gb;
      int kcur[YY_U], pcur[YY_U], kn[YY_U], pn[YY_U];
      load_kp(e0, kpn);
#pragma unroll
      for (int u = 0; u < YY_U; u++) { kcur[u] = kpn.k[u]; pcur[u] = kpn.p[u]; }
      gather(kpn, ga);
      load_kp(e0 + 32 * YY_U, kpnn);
      for (int32_t e = e0; e < e1; e += 32 * YY_U) {
        const bool more = (e + 32 * YY_U) < e1;
        if (more) {
#pragma unroll
          for (int u = 0; u < YY_U; u++) { kn[u] = kpnn.k[u]; pn[u] = kpnn.p[u]; }
          gather(kpnn, gb);
          load_kp(e + 64 * YY_U, kpnn);
        }
        double tt[YY_U];
#pragma unroll
        for (int u = 0; u < YY_U; u++) {
          tt[u] = ga.vs[u][0] * ga.wk[u];
          rsum += tt[u] * ga.rr[u];
        }
        // s = 0: the diagonal (c1 == c) -- every lane hits it: warp sum, no scatter
#pragma unroll
        for (int u = 0; u < YY_U; u++) diag += tt[u] * ga.vs[u][0];
        // s >= 1: off-diagonal scatter into the private column
#pragma unroll
        for (int u = 0; u < YY_U; u++) {
#pragma unroll
          for (int s2 = 1; s2 < YY_SMAX; s2++) {
            int64_t c1 = -1;
            if (s2 < ga.l[u]) {
              c1 = (int64_t)ga.cs[u][s2] - c - base;
              if (c1 < 0 || c1 >= clen) c1 = -1;
            }
            const bool go = c1 >= 0;
            const unsigned gomask = __ballot_sync(0xffffffffu, go);
            if (gomask == 0u) continue;
            const double upd = tt[u] * ga.vs[u][s2];
            if (go) {
#ifdef MDS_YY_NOMATCH
              const unsigned peers = 1u << lane;   // timing experiment only (wrong on collisions)
#else
              const unsigned peers = __match_any_sync(gomask, (int)c1);
#endif
              if (peers == (1u << lane)) {
                acc[c1] -= upd;
              } else {
                const int rank = __popc(peers & lanemask_lt);
                const int gs = __popc(peers);
                for (int qq = 0; qq < gs; qq++) {
                  if (rank == qq) acc[c1] -= upd;
                  __syncwarp(peers);
                }
              }
            }
            __syncwarp();
          }
          // rare: suffix longer than YY_SMAX
          for (int s2 = YY_SMAX; __any_sync(0xffffffffu, s2 < ga.l[u]); s2++) {
            int64_t c1 = -1;
            double upd = 0.0;
            if (s2 < ga.l[u]) {
              c1 = (int64_t)colidx[pcur[u] + s2] - c - base;
              upd = tt[u] * val[pcur[u] + s2];
              if (c1 < 0 || c1 >= clen) c1 = -1;
            }
            const bool go = c1 >= 0;
            const unsigned gomask = __ballot_sync(0xffffffffu, go);
            if (go) {
              const unsigned peers = __match_any_sync(gomask, (int)c1);
              const int rank = __popc(peers & lanemask_lt);
              const int gs = __popc(peers);
              for (int qq = 0; qq < gs; qq++) {
                if (rank == qq) acc[c1] -= upd;
                __syncwarp(peers);
              }
            }
            __syncwarp();
          }
        }
        if (more) {
          ga = gb;
#pragma unroll
          for (int u = 0; u < YY_U; u++) { kcur[u] = kn[u]; pcur[u] = pn[u]; }
        }
      }
      (void)kcur;
      diag = warp_sum(diag);
      __syncwarp();
      // diagonal terms -diag(0_{m_E}, 1/d_h) - delta_c I, then one coalesced column write
      double* Mc = M + (n_d + c) * ldm + n_d + c + base;
      for (int64_t i = lane; i < clen; i += 32) {
        double v = acc[i];
        if (base + i == 0) {
          v = -diag - delta_c;
          if (c >= m_E) {
            const double dh = d_h[c - m_E];
            if (!(dh > 0.0)) mds_set_status(status, MDS_ERR_NONPOSITIVE);
            v = v - 1.0 / dh;
          }
        }
        stg_ef(Mc + i, v);
      }
      __syncwarp();
    }
    if (rhs_c && r) {
      rsum = warp_sum(rsum);
      if (lane == 0) rhs_c[n_d + c] = r[n_s + n_d + c] - rsum;
    }
  }
}

extern "C" int mds_condense(const mds_plan* P, const double* js_val, const double* h_ss, const double* sigma_s,
                            const double* H_dd, int64_t ldh, const double* sigma_d, const double* J_d, int64_t ldj,
                            const double* d_h, double delta_w, double delta_c, const double* r,
                            double* M, int64_t ldm, double* rhs_c, double* w_out, int32_t* status, void* stream) {
  if (!P) return MDS_ERR_ARG;
  const int64_t n_s = P->n_s, n_d = P->n_d, m = P->m_E + P->m_I, N = n_d + m;
  if (N == 0) return MDS_OK;
  if (!M || ldm < N) return MDS_ERR_ARG;
  if (n_s > 0 && (!h_ss || !sigma_s || !w_out || (P->nnz > 0 && !js_val))) return MDS_ERR_ARG;
  if (n_d > 0 && (!H_dd || ldh < n_d || !sigma_d)) return MDS_ERR_ARG;
  if (n_d > 0 && m > 0 && (!J_d || ldj < m)) return MDS_ERR_ARG;
  if (P->m_I > 0 && !d_h) return MDS_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  if (rhs_c && !r) rhs_c = nullptr;
  if (n_s > 0) {
    int64_t blocks = std::min<int64_t>(mds_cdiv(n_s, 256), 148 * 16);
    MDS_LAUNCH(PC_CONDENSE_W, st,
               MDS_CUDA_TRY(launch_pdl(k_condense_w, dim3((unsigned)blocks), dim3(256), 0, st, n_s, h_ss, sigma_s, delta_w,
                                       w_out, status)));
  }
  if (m > 0) {
    // warp-private accumulator columns: <= 4096 doubles each; warps per CTA sized to ~192 KB
    // (MDS_YY_ACC caps the column window: longer columns take several passes over their list,
    //  in exchange for more resident warps; A/B knob)
    static const int64_t acc_cap = std::getenv("MDS_YY_ACC") ? std::atoll(std::getenv("MDS_YY_ACC")) : 4096;
    const int64_t acc_len = std::min<int64_t>(((m + 31) / 32) * 32, acc_cap);
    static bool attr_set = false;
    if (!attr_set) {
      cudaFuncSetAttribute(k_condense_yy<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * 4096 * 8);
      cudaFuncSetAttribute(k_condense_yy<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 2048 * 8);
      cudaFuncSetAttribute(k_condense_yy<12>, cudaFuncAttributeMaxDynamicSharedMemorySize, 12 * 2048 * 8);
      (void)cudaGetLastError();
      attr_set = true;
    }
    const int64_t ntask = (m + 1) / 2;
    if (acc_len > 2048) {
      constexpr int W = 6;
      size_t smem = sizeof(double) * acc_len * W;
      MDS_LAUNCH(PC_CONDENSE_YY, st,
                 MDS_CUDA_TRY(launch_pdl(k_condense_yy<W>, dim3((unsigned)mds_cdiv(ntask, W)), dim3(W * 32), smem, st,
                     n_d, P->m_E, m, acc_len, P->rowptr, P->colidx, js_val, P->tptr, P->tkp, w_out, d_h, delta_c,
                     r, n_s, M, ldm, rhs_c, status)));
    } else if (acc_len == 2048 && m > 2048) {
      constexpr int W = 12;
      size_t smem = sizeof(double) * acc_len * W;
      MDS_LAUNCH(PC_CONDENSE_YY, st,
                 MDS_CUDA_TRY(launch_pdl(k_condense_yy<W>, dim3((unsigned)mds_cdiv(ntask, W)), dim3(W * 32), smem, st,
                     n_d, P->m_E, m, acc_len, P->rowptr, P->colidx, js_val, P->tptr, P->tkp, w_out, d_h, delta_c,
                     r, n_s, M, ldm, rhs_c, status)));
    } else {
      constexpr int W = 8;
      size_t smem = sizeof(double) * acc_len * W;
      MDS_LAUNCH(PC_CONDENSE_YY, st,
                 MDS_CUDA_TRY(launch_pdl(k_condense_yy<W>, dim3((unsigned)mds_cdiv(ntask, W)), dim3(W * 32), smem, st,
                     n_d, P->m_E, m, acc_len, P->rowptr, P->colidx, js_val, P->tptr, P->tkp, w_out, d_h, delta_c,
                     r, n_s, M, ldm, rhs_c, status)));
    }
  }
  // dense blocks after (and concurrently with) k_condense_yy; see k_condense_dense
  if (n_d > 0) {
    int64_t blocks = std::min<int64_t>(n_d, 148 * 8);
    MDS_LAUNCH(PC_CONDENSE_DENSE, st,
               MDS_CUDA_TRY(launch_pdl(k_condense_dense, dim3((unsigned)blocks), dim3(256), 0, st, n_d, m, H_dd, ldh, sigma_d,
                                       delta_w, J_d, ldj, M, ldm, r ? r + n_s : nullptr, rhs_c)));
  }
  return MDS_OK;
}
