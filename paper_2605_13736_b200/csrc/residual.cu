// residual.cu — mds_kkt_residual: out = b - K x for the FULL (uncondensed)
// Eq.(5) system of PAPER.md:147-159, the mixed sparse/dense mat-vec class K2
// of PAPER.md:185 ("K2 ... mixed dense-sparse matrix-vector products").
//   K = [ Q_s        0          J_s        ]   Q_s = diag(h_ss + sigma_s + delta_w)
//       [ 0          Q_d        J_d^T      ]   Q_d = H_dd + diag(sigma_d) + delta_w I
//       [ J_s^T      J_d       -D_y        ]   D_y = diag(0_{m_E}, 1/d_h) + delta_c I
// (rows = sparse variables x_s | dense variables x_d | constraints y = (y_g, y_h);
//  J_s is n_s x m (reading R1), J_d is m x n_d.)
// Kernels (HBM-bound; every entry of the lower H_dd and of J_d is read ONCE):
//   k_res_s     x_s rows: q_k x_s[k] + sum_c J_s[k,c] y[c]          (thread per sparse row, CSR)
//   k_res_y     (J_s^T x_s)[c] (constraint-major transpose list of the plan, fixed order; warp per constraint)
//   k_res_tiles one CTA per 64 x 64 tile of the lower H_dd and of J_d: row sums and (transposed)
//               column sums of the tile into per-tile partial slots (H x_d, J_d x_d, J_d^T y)
//   k_res_final x_d rows ((sigma_d+delta_w) x_d + the H / J_d^T slots in slot order) and y rows
//               (J_s^T x_s + the J_d slots - D_y y)
//   k_res_norm  ||out||_inf (fixed-order two-level max)
#include <algorithm>

#include "common.cuh"

const int32_t* mds_plan_rowptr(const mds_plan* P);
const int32_t* mds_plan_colidx(const mds_plan* P);
const int32_t* mds_plan_tptr(const mds_plan* P);
const int2* mds_plan_tkp(const mds_plan* P);

namespace {
constexpr unsigned TKP_PMASK_R = (1u << 27) - 1u;

__global__ void k_res_s(int64_t n_s, int64_t n_d, const int32_t* __restrict__ rowptr,
                        const int32_t* __restrict__ colidx, const double* __restrict__ val,
                        const double* __restrict__ h_ss, const double* __restrict__ sigma_s, double delta_w,
                        const double* __restrict__ x, const double* __restrict__ b, double* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const double* y = x + n_s + n_d;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n_s; k += (int64_t)gridDim.x * blockDim.x) {
    double v = (h_ss[k] + sigma_s[k] + delta_w) * x[k];
    for (int32_t p = rowptr[k]; p < rowptr[k + 1]; p++) v += val[p] * y[colidx[p]];
    out[k] = b ? b[k] - v : v;
  }
}

// The dense blocks, one CTA per 64 x 64 tile, every dense entry read ONCE:
//   tiles [0, nth):        lower tiles (I >= J) of H_dd -- row sums (H x_d) into y_d block I,
//                          for I > J column sums (the transposed upper half) into y_d block J;
//                          a diagonal tile adds its strictly lower part transposed
//   tiles [nth, nth+ntj):  tiles (C, J) of J_d -- row sums (J_d x_d) into y block C,
//                          column sums (J_d^T y) into y_d block J
// Each partial (64 values) goes to its own slot; k_res_final adds the slots of an
// output block in slot order (deterministic).  Slots of y_d block b: [0, nbd) H row
// parts from tile (b, J) / column parts from tile (I, b), nbd: the diagonal tile's
// transposed part, nbd + 1 + C: J_d tile (C, b); of y block C: J = 0 .. nbd-1.
constexpr int RT = 64;
struct ResTiles {
  int64_t n_d, m, nbd, nbm, nth;
  const double* H; int64_t ldh;
  const double* Jd; int64_t ldj;
  const double* xd;   // [n_d]
  const double* y;    // [m]
  double* pd;         // [nbd][nbd + 1 + nbm][64]
  double* py;         // [nbm][nbd][64]
};
__device__ __forceinline__ void tri_ij(int64_t t, int64_t& I, int64_t& J) {
  I = (int64_t)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
  while (I * (I + 1) / 2 > t) I--;
  while ((I + 1) * (I + 2) / 2 <= t) I++;
  J = t - I * (I + 1) / 2;
}

__global__ void __launch_bounds__(256) k_res_tiles(ResTiles a) {
  pdl_wait();
  pdl_trigger();
  __shared__ double xr[RT], xc[RT];     // the vector pieces for row sums (x_J) and column sums (x_I)
  __shared__ double rp[8][RT];          // per-warp row partials
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t t = blockIdx.x;
  const bool isH = t < a.nth;
  int64_t I, J;
  if (isH) tri_ij(t, I, J);
  else { I = (t - a.nth) / a.nbd; J = (t - a.nth) % a.nbd; }
  const int64_t r0 = I * RT, c0 = J * RT;
  const int64_t nrow = isH ? a.n_d : a.m;
  const double* A = isH ? a.H : a.Jd;
  const int64_t ld = isH ? a.ldh : a.ldj;
  if (threadIdx.x < RT) {
    const int64_t c = c0 + threadIdx.x, r = r0 + threadIdx.x;
    xr[threadIdx.x] = (c < a.n_d) ? a.xd[c] : 0.0;
    xc[threadIdx.x] = isH ? ((r < a.n_d) ? a.xd[r] : 0.0) : ((r < a.m) ? a.y[r] : 0.0);
  }
  __syncthreads();
  const bool diag = isH && I == J;
  double s0 = 0.0, s1 = 0.0;   // row sums of rows lane, lane + 32 over this warp's 8 columns
#pragma unroll
  for (int u = 0; u < 8; u++) {
    const int cl = warp * 8 + u;
    const int64_t c = c0 + cl;
    double v0 = 0.0, v1 = 0.0;
    if (c < a.n_d) {
      const int64_t ra = r0 + lane, rb = r0 + lane + 32;
      if (ra < nrow && (!diag || lane >= cl)) v0 = A[ra + c * ld];
      if (rb < nrow && (!diag || lane + 32 >= cl)) v1 = A[rb + c * ld];
    }
    s0 = fma(v0, xr[cl], s0);
    s1 = fma(v1, xr[cl], s1);
    // column sum (transposed part): the whole tile, or the strictly lower part of a diagonal tile
    double cs = (diag ? (lane > cl ? v0 : 0.0) * xc[lane] + (lane + 32 > cl ? v1 : 0.0) * xc[lane + 32]
                      : v0 * xc[lane] + v1 * xc[lane + 32]);
    cs = warp_sum(cs);
    if (lane == 0 && (!isH || I > J || diag)) {
      double* dst = isH ? a.pd + ((J * (a.nbd + 1 + a.nbm)) + (diag ? a.nbd : I)) * RT
                        : a.pd + ((J * (a.nbd + 1 + a.nbm)) + a.nbd + 1 + I) * RT;
      dst[cl] = cs;
    }
  }
  rp[warp][lane] = s0;
  rp[warp][lane + 32] = s1;
  __syncthreads();
  if (threadIdx.x < RT) {
    double v = 0.0;
#pragma unroll
    for (int w = 0; w < 8; w++) v += rp[w][threadIdx.x];
    double* dst = isH ? a.pd + ((I * (a.nbd + 1 + a.nbm)) + J) * RT : a.py + (I * a.nbd + J) * RT;
    dst[threadIdx.x] = v;
  }
}

// x_d rows and y rows: the dense partials in slot order plus the diagonal / sparse terms
__global__ void __launch_bounds__(256) k_res_final(int64_t n_s, int64_t n_d, int64_t m_E, int64_t m, ResTiles a,
                                                   const double* __restrict__ sigma_d, double delta_w,
                                                   const double* __restrict__ d_h, double delta_c,
                                                   const double* __restrict__ ys, const double* __restrict__ x,
                                                   const double* __restrict__ b, double* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n_d) {
    const int64_t bb = i / RT, e = i % RT, ns = a.nbd + 1 + a.nbm;
    const double* p = a.pd + bb * ns * RT + e;
    double v0 = 0.0, v1 = 0.0, v2 = 0.0, v3 = 0.0;   // four interleaved partial sums (fixed order)
    int64_t sl = 0;
    for (; sl + 4 <= ns; sl += 4) {
      v0 += p[sl * RT]; v1 += p[(sl + 1) * RT]; v2 += p[(sl + 2) * RT]; v3 += p[(sl + 3) * RT];
    }
    for (; sl < ns; sl++) v0 += p[sl * RT];
    double v = (v0 + v1) + (v2 + v3);
    v += (sigma_d[i] + delta_w) * x[n_s + i];
    const int64_t o = n_s + i;
    out[o] = b ? b[o] - v : v;
  } else if (i < n_d + m) {
    const int64_t c = i - n_d, cb = c / RT, e = c % RT;
    const double* p = a.py + cb * a.nbd * RT + e;
    double v0 = 0.0, v1 = 0.0, v2 = 0.0, v3 = 0.0;
    int64_t sl = 0;
    for (; sl + 4 <= a.nbd; sl += 4) {
      v0 += p[sl * RT]; v1 += p[(sl + 1) * RT]; v2 += p[(sl + 2) * RT]; v3 += p[(sl + 3) * RT];
    }
    for (; sl < a.nbd; sl++) v0 += p[sl * RT];
    double v = ys[c] + ((v0 + v1) + (v2 + v3));
    const double yc = x[n_s + n_d + c];
    const double dy = (c >= m_E ? 1.0 / d_h[c - m_E] : 0.0) + delta_c;
    v -= dy * yc;
    const int64_t o = n_s + n_d + c;
    out[o] = b ? b[o] - v : v;
  }
}

// (J_s^T x_s)[c] per constraint (constraint-major transpose list of the plan, fixed order)
__global__ void k_res_y(int64_t m, const int32_t* __restrict__ tptr, const int2* __restrict__ tkp,
                        const double* __restrict__ val, const double* __restrict__ x, double* __restrict__ ys) {
  pdl_wait();
  pdl_trigger();
  const int lane = threadIdx.x & 31;
  const int64_t c = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (c >= m) return;
  constexpr int U = 4;   // independent entries (gathers) in flight per lane
  double acc[U];
#pragma unroll
  for (int u = 0; u < U; u++) acc[u] = 0.0;
  const int32_t e1 = tptr[c + 1];
  for (int32_t e = tptr[c] + lane; e < e1; e += 32 * U) {
    int2 kp[U];
#pragma unroll
    for (int u = 0; u < U; u++) kp[u] = (e + 32 * u < e1) ? tkp[e + 32 * u] : make_int2(-1, 0);
    double pv[U], xv[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      pv[u] = (kp[u].x >= 0) ? val[(unsigned)kp[u].y & TKP_PMASK_R] : 0.0;
      xv[u] = (kp[u].x >= 0) ? x[kp[u].x] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; u++) acc[u] = fma(pv[u], xv[u], acc[u]);
  }
  const double v = warp_sum((acc[0] + acc[1]) + (acc[2] + acc[3]));
  if (lane == 0) ys[c] = v;
}

__global__ void __launch_bounds__(1024) k_res_norm(int64_t n, const double* __restrict__ v, double* out) {
  pdl_wait();
  pdl_trigger();
  double a = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) a = fmax(a, fabs(v[i]));
  a = warp_max(a);
  __shared__ double sh[32];
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = a;
  __syncthreads();
  if (threadIdx.x == 0) {
    double r = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); w++) r = fmax(r, sh[w]);
    *out = r;
  }
}
}  // namespace

namespace {
struct ResLayout {
  size_t ys, pd, py, total;
};
ResLayout res_layout(int64_t n_d, int64_t m) {
  const int64_t nbd = (n_d + RT - 1) / RT, nbm = (m + RT - 1) / RT;
  ResLayout L;
  L.ys = 0;
  L.pd = (size_t)std::max<int64_t>(m, 1) * 8;
  L.pd = (L.pd + 255) / 256 * 256;
  L.py = L.pd + (size_t)nbd * (nbd + 1 + nbm) * RT * 8;
  L.total = L.py + (size_t)nbm * nbd * RT * 8 + 8;
  return L;
}
}  // namespace

extern "C" size_t mds_kkt_residual_workspace_size(const mds_plan* P) {
  if (!P) return 0;
  int64_t d[5];
  mds_plan_dims(P, d);
  return res_layout(d[1], d[2] + d[3]).total;
}

extern "C" int mds_kkt_residual(const mds_plan* P, const double* js_val, const double* h_ss, const double* sigma_s,
                                const double* H_dd, int64_t ldh, const double* sigma_d, const double* J_d, int64_t ldj,
                                const double* d_h, double delta_w, double delta_c, const double* x, const double* b,
                                double* out, double* rnorm, void* work, size_t work_bytes, void* stream) {
  if (!P || !x || !out) return MDS_ERR_ARG;
  int64_t d[5];
  mds_plan_dims(P, d);
  const int64_t n_s = d[0], n_d = d[1], m_E = d[2], m_I = d[3], nnz = d[4], m = m_E + m_I;
  if (n_s > 0 && (!h_ss || !sigma_s || (nnz > 0 && !js_val))) return MDS_ERR_ARG;
  if (n_d > 0 && (!H_dd || ldh < n_d || !sigma_d)) return MDS_ERR_ARG;
  if (n_d > 0 && m > 0 && (!J_d || ldj < m)) return MDS_ERR_ARG;
  if (m_I > 0 && !d_h) return MDS_ERR_ARG;
  const ResLayout L = res_layout(n_d, m);
  if (!work || work_bytes < L.total) return MDS_ERR_WORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  char* base = reinterpret_cast<char*>(work);
  double* ys = reinterpret_cast<double*>(base + L.ys);
  ResTiles a;
  a.n_d = n_d; a.m = m; a.nbd = (n_d + RT - 1) / RT; a.nbm = (m + RT - 1) / RT; a.nth = a.nbd * (a.nbd + 1) / 2;
  a.H = H_dd; a.ldh = ldh; a.Jd = J_d; a.ldj = ldj; a.xd = x + n_s; a.y = x + n_s + n_d;
  a.pd = reinterpret_cast<double*>(base + L.pd);
  a.py = reinterpret_cast<double*>(base + L.py);
  if (n_s > 0)
    MDS_CUDA_TRY(launch_pdl(k_res_s, dim3((unsigned)std::min<int64_t>(mds_cdiv(n_s, 256), 148 * 16)), dim3(256), 0, st,
                            n_s, n_d, mds_plan_rowptr(P), mds_plan_colidx(P), js_val, h_ss, sigma_s, delta_w, x, b,
                            out));
  if (m > 0) {
    if (n_s > 0)
      MDS_CUDA_TRY(launch_pdl(k_res_y, dim3((unsigned)mds_cdiv(m * 32, 256)), dim3(256), 0, st, m, mds_plan_tptr(P),
                              mds_plan_tkp(P), js_val, x, ys));
    else
      MDS_CUDA_TRY(cudaMemsetAsync(ys, 0, sizeof(double) * m, st));
  }
  if (n_d > 0) {
    const int64_t ntiles = a.nth + (m > 0 ? a.nbm * a.nbd : 0);
    MDS_CUDA_TRY(launch_pdl(k_res_tiles, dim3((unsigned)ntiles), dim3(256), 0, st, a));
  }
  if (n_d + m > 0)
    MDS_CUDA_TRY(launch_pdl(k_res_final, dim3((unsigned)mds_cdiv(n_d + m, 256)), dim3(256), 0, st, n_s, n_d, m_E, m, a,
                            sigma_d, delta_w, d_h, delta_c, (const double*)ys, x, b, out));
  if (rnorm) MDS_CUDA_TRY(launch_pdl(k_res_norm, dim3(1), dim3(1024), 0, st, n_s + n_d + m, (const double*)out, rnorm));
  return MDS_OK;
}
