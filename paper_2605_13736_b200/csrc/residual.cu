// residual.cu — mds_kkt_residual: out = b - K x for the FULL (uncondensed)
// Eq.(5) system of PAPER.md:147-159, the mixed sparse/dense mat-vec class K2
// of PAPER.md:185 ("K2 ... mixed dense-sparse matrix-vector products").
//   K = [ Q_s        0          J_s        ]   Q_s = diag(h_ss + sigma_s + delta_w)
//       [ 0          Q_d        J_d^T      ]   Q_d = H_dd + diag(sigma_d) + delta_w I
//       [ J_s^T      J_d       -D_y        ]   D_y = diag(0_{m_E}, 1/d_h) + delta_c I
// (rows = sparse variables x_s | dense variables x_d | constraints y = (y_g, y_h);
//  J_s is n_s x m (reading R1), J_d is m x n_d.)
// Kernels (HBM-bound; H_dd and J_d are each read twice, once per orientation):
//   k_res_s   x_s rows: q_k x_s[k] + sum_c J_s[k,c] y[c]            (thread per sparse row, CSR)
//   k_res_y   y rows:   sum_k J_s[k,c] x_s[k] (constraint-major transpose
//                       list of the plan, fixed order) + (J_d x_d)[c] - D_y[c] y[c]   (warp per constraint)
//   k_res_jd  (J_d x_d)[c] for all c                                 (thread per constraint, coalesced columns)
//   k_res_d   x_d rows: column part sum_{j>=i} H[j,i] x[j], row part sum_{j<i} H[i,j] x[j] (lower storage),
//                       (sigma_d+delta_w) x_d[i], (J_d^T y)[i]       (warp per dense variable)
//   k_res_norm ||out||_inf (fixed-order two-level max)
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

__global__ void k_res_jd(int64_t m, int64_t n_d, const double* __restrict__ Jd, int64_t ldj,
                         const double* __restrict__ xd, double* __restrict__ jx) {
  pdl_wait();
  pdl_trigger();
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < m; c += (int64_t)gridDim.x * blockDim.x) {
    double v = 0.0;
    for (int64_t j = 0; j < n_d; j++) v += Jd[c + j * ldj] * xd[j];
    jx[c] = v;
  }
}

__global__ void k_res_y(int64_t n_s, int64_t n_d, int64_t m_E, int64_t m, const int32_t* __restrict__ tptr,
                        const int2* __restrict__ tkp, const double* __restrict__ val, const double* __restrict__ d_h,
                        double delta_c, const double* __restrict__ jx, const double* __restrict__ x,
                        const double* __restrict__ b, double* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const int lane = threadIdx.x & 31;
  const int64_t c = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (c >= m) return;
  double v = 0.0;
  for (int32_t e = tptr[c] + lane; e < tptr[c + 1]; e += 32) {
    const int2 kp = tkp[e];
    v += val[(unsigned)kp.y & TKP_PMASK_R] * x[kp.x];
  }
  v = warp_sum(v);
  if (lane == 0) {
    const double yc = x[n_s + n_d + c];
    const double dy = (c >= m_E ? 1.0 / d_h[c - m_E] : 0.0) + delta_c;
    v += jx[c] - dy * yc;
    const int64_t o = n_s + n_d + c;
    out[o] = b ? b[o] - v : v;
  }
}

__global__ void k_res_d(int64_t n_s, int64_t n_d, int64_t m, const double* __restrict__ H, int64_t ldh,
                        const double* __restrict__ sigma_d, double delta_w, const double* __restrict__ Jd,
                        int64_t ldj, const double* __restrict__ x, const double* __restrict__ b,
                        double* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const int lane = threadIdx.x & 31;
  const int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (i >= n_d) return;
  const double* xd = x + n_s;
  const double* y = x + n_s + n_d;
  double v = 0.0;
  for (int64_t j = i + lane; j < n_d; j += 32) v += H[j + i * ldh] * xd[j];          // column i, j >= i
  for (int64_t j = lane; j < i; j += 32) v += H[i + j * ldh] * xd[j];                // row i, j < i
  for (int64_t c = lane; c < m; c += 32) v += Jd[c + i * ldj] * y[c];                // (J_d^T y)_i
  v = warp_sum(v);
  if (lane == 0) {
    v += (sigma_d[i] + delta_w) * xd[i];
    const int64_t o = n_s + i;
    out[o] = b ? b[o] - v : v;
  }
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

extern "C" size_t mds_kkt_residual_workspace_size(int64_t m) { return sizeof(double) * (size_t)std::max<int64_t>(m, 1); }

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
  if (m > 0 && (!work || work_bytes < mds_kkt_residual_workspace_size(m))) return MDS_ERR_WORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  double* jx = reinterpret_cast<double*>(work);
  if (n_s > 0)
    MDS_CUDA_TRY(launch_pdl(k_res_s, dim3((unsigned)std::min<int64_t>(mds_cdiv(n_s, 256), 148 * 16)), dim3(256), 0, st,
                            n_s, n_d, mds_plan_rowptr(P), mds_plan_colidx(P), js_val, h_ss, sigma_s, delta_w, x, b,
                            out));
  if (m > 0) {
    if (n_d > 0)
      MDS_CUDA_TRY(launch_pdl(k_res_jd, dim3((unsigned)mds_cdiv(m, 128)), dim3(128), 0, st, m, n_d, J_d, ldj,
                              x + n_s, jx));
    else
      MDS_CUDA_TRY(cudaMemsetAsync(jx, 0, sizeof(double) * m, st));
    MDS_CUDA_TRY(launch_pdl(k_res_y, dim3((unsigned)mds_cdiv(m * 32, 256)), dim3(256), 0, st, n_s, n_d, m_E, m,
                            mds_plan_tptr(P), mds_plan_tkp(P), js_val, d_h, delta_c, (const double*)jx, x, b, out));
  }
  if (n_d > 0)
    MDS_CUDA_TRY(launch_pdl(k_res_d, dim3((unsigned)mds_cdiv(n_d * 32, 256)), dim3(256), 0, st, n_s, n_d, m, H_dd, ldh,
                            sigma_d, delta_w, J_d, ldj, x, b, out));
  if (rnorm) MDS_CUDA_TRY(launch_pdl(k_res_norm, dim3(1), dim3(1024), 0, st, n_s + n_d + m, (const double*)out, rnorm));
  return MDS_OK;
}
