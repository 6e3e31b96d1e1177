// ipm.cu — the vector kernels of the interior-point loop around the hot path
// (K1 of PAPER.md:184: "vector-vector axpy operations" and the reductions of
// the filter line search), for the convex-QP IPM of
// DESIGN.md reading R23.  All elementwise / fixed-order reductions; HBM-bound.
//
// Layout (one iterate): P = [x_s | x_d | s] (n + m_I), lo/up over P (the slack
// bounds h_l/h_u in the tail; |b| >= 1e20 infinite), bound duals zl/zu over P
// (the slack duals v_l/v_u in the tail), y = (y_g, y_h) (m).  Kxy = (H x + J^T y,
// J x) is mds_kkt_residual's K x with sigma = delta = 0 and D_y = 0.
#include <algorithm>

#include "common.cuh"

namespace {
constexpr int IT = 256;        // threads per CTA
constexpr int NOUT = 8;        // reduction outputs per call

__device__ __forceinline__ bool fin(double b) { return fabs(b) < MDS_INF_BOUND; }

struct IpmDims {
  int64_t n, m_E, m_I;         // n = n_s + n_d
};

// ---------------------------------------------------------------------------
// rhs: sigma, the Eq.(5) right-hand side r = (r_x, r_y), q, residuals.
//   sigma_i  = zl/(P-lo) + zu/(up-P)   (finite terms; the slack tail is D_h)
//   r_x      = -(Kxy_x + c - mu/(x-lo) + mu/(up-x))
//   r_yE     = -(J_E x - g_E)
//   q        = y_h + mu/(s-h_l) - mu/(h_u-s)
//   r_yI     = -(J_I x - s) + q / D_h
//   res_d    = (Kxy_x + c - zl + zu ; -y_h - v_l + v_u),  res_p = (J_E x - g_E ; J_I x - s)
__global__ void __launch_bounds__(IT) k_ipm_rhs(IpmDims d, const double* __restrict__ Kxy, const double* __restrict__ c,
                                                const double* __restrict__ g_E, const double* __restrict__ P,
                                                const double* __restrict__ lo, const double* __restrict__ up,
                                                const double* __restrict__ zl, const double* __restrict__ zu,
                                                const double* __restrict__ y, double mu, double* __restrict__ sigma,
                                                double* __restrict__ r, double* __restrict__ q,
                                                double* __restrict__ res_d, double* __restrict__ res_p) {
  pdl_wait();
  pdl_trigger();
  const int64_t np = d.n + d.m_I;
  for (int64_t i = blockIdx.x * (int64_t)IT + threadIdx.x; i < np; i += (int64_t)gridDim.x * IT) {
    const double v = P[i], l = lo[i], u = up[i];
    const bool hl = fin(l), hu = fin(u);
    const double gl = hl ? v - l : 1.0, gu = hu ? u - v : 1.0;
    const double sg = (hl ? zl[i] / gl : 0.0) + (hu ? zu[i] / gu : 0.0);
    const double bl = hl ? mu / gl : 0.0, bu = hu ? mu / gu : 0.0;
    sigma[i] = sg;
    if (i < d.n) {
      const double gx = Kxy[i] + c[i];
      r[i] = -(gx - (bl - bu));
      res_d[i] = gx - zl[i] + zu[i];
    } else {
      const int64_t j = i - d.n;                    // inequality j
      const double yh = y[d.m_E + j];
      const double qj = yh + bl - bu;
      q[j] = qj;
      const double rp = Kxy[d.n + d.m_E + j] - v;   // J_I x - s
      res_p[d.m_E + j] = rp;
      r[d.n + d.m_E + j] = -rp + qj / sg;
      res_d[i] = -yh - zl[i] + zu[i];
    }
  }
  for (int64_t j = blockIdx.x * (int64_t)IT + threadIdx.x; j < d.m_E; j += (int64_t)gridDim.x * IT) {
    const double rp = Kxy[d.n + j] - g_E[j];
    res_p[j] = rp;
    r[d.n + j] = -rp;
  }
}

// directions: dP = (dx, ds), ds = (dy_h + q)/D_h; dzl = mu/gl - zl - (zl/gl) dP; dzu = mu/gu - zu + (zu/gu) dP.
// Also dx0 = (dx, 0) for the K0 product of the line search.
__global__ void __launch_bounds__(IT) k_ipm_dir(IpmDims d, const double* __restrict__ dxy, const double* __restrict__ q,
                                                const double* __restrict__ sigma, const double* __restrict__ P,
                                                const double* __restrict__ lo, const double* __restrict__ up,
                                                const double* __restrict__ zl, const double* __restrict__ zu, double mu,
                                                double* __restrict__ dP, double* __restrict__ dzl,
                                                double* __restrict__ dzu, double* __restrict__ dx0) {
  pdl_wait();
  pdl_trigger();
  const int64_t np = d.n + d.m_I;
  for (int64_t i = blockIdx.x * (int64_t)IT + threadIdx.x; i < np; i += (int64_t)gridDim.x * IT) {
    double dv;
    if (i < d.n) {
      dv = dxy[i];
      dx0[i] = dv;
    } else {
      const int64_t j = i - d.n;
      dv = (dxy[d.n + d.m_E + j] + q[j]) / sigma[i];
    }
    dP[i] = dv;
    const double v = P[i], l = lo[i], u = up[i];
    const bool hl = fin(l), hu = fin(u);
    const double gl = hl ? v - l : 1.0, gu = hu ? u - v : 1.0;
    dzl[i] = hl ? mu / gl - zl[i] - (zl[i] / gl) * dv : 0.0;
    dzu[i] = hu ? mu / gu - zu[i] + (zu[i] / gu) * dv : 0.0;
  }
}

// ---------------------------------------------------------------------------
// Reductions (fixed order: per-thread grid-stride partials, warp xor trees, CTA
// partials, the last CTA combines the CTA partials in index order).
//   mode 0 (errors):   out = [||res_d||_inf, ||res_p||_inf, max gap z, max |gap z - mu|]
//   mode 1 (scalars):  out = [f0 = 1/2 x.Kxy_x - 1/2 y.Kxy_y + c.x, gdx = Kxy_x.dx - y.Kd_y + c.dx,
//                             dHd = dx.Kd_x, gphi_b = -(b_l - b_u).dP (barrier part of grad phi . d),
//                             theta0 = ||res_p||_1, B0 = sum log gaps]
//   mode 2 (trial a):  out = [theta(a) = ||res_p + a dr_p||_1, B(a) = sum log gaps(P + a dP)],
//                      dr_p = Kd_y - (0, ds)
struct RedIn {
  const double *P, *dP, *lo, *up, *zl, *zu, *y, *c, *Kxy, *Kd, *res_d, *res_p;
  double mu, alpha;
};

__device__ __forceinline__ double wred(double v, bool mx) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double w = __shfl_xor_sync(0xffffffffu, v, o);
    v = mx ? fmax(v, w) : v + w;
  }
  return v;
}

template <int MODE>
__global__ void __launch_bounds__(IT) k_ipm_reduce(IpmDims d, RedIn a, double* __restrict__ partials,
                                                   unsigned* counter, double* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  constexpr int NV = MODE == 0 ? 4 : MODE == 1 ? 6 : 2;
  constexpr bool IS_MAX[3][6] = {{true, true, true, true, false, false},
                                 {false, false, false, false, false, false},
                                 {false, false, false, false, false, false}};
  double acc[NV];
#pragma unroll
  for (int k = 0; k < NV; k++) acc[k] = 0.0;
  const int64_t np = d.n + d.m_I, m = d.m_E + d.m_I;
  const int64_t t0 = blockIdx.x * (int64_t)IT + threadIdx.x, ts = (int64_t)gridDim.x * IT;
  for (int64_t i = t0; i < np; i += ts) {
    const double l = a.lo[i], u = a.up[i];
    const bool hl = fin(l), hu = fin(u);
    if (MODE == 0) {
      const double v = a.P[i];
      acc[0] = fmax(acc[0], fabs(a.res_d[i]));
      if (hl) {
        const double cz = (v - l) * a.zl[i];
        acc[2] = fmax(acc[2], fabs(cz));
        acc[3] = fmax(acc[3], fabs(cz - a.mu));
      }
      if (hu) {
        const double cz = (u - v) * a.zu[i];
        acc[2] = fmax(acc[2], fabs(cz));
        acc[3] = fmax(acc[3], fabs(cz - a.mu));
      }
    } else if (MODE == 1) {
      const double v = a.P[i], dv = a.dP[i];
      const double gl = hl ? v - l : 1.0, gu = hu ? u - v : 1.0;
      const double bl = hl ? a.mu / gl : 0.0, bu = hu ? a.mu / gu : 0.0;
      if (i < d.n) {
        acc[0] += 0.5 * v * a.Kxy[i] + a.c[i] * v;
        acc[1] += (a.Kxy[i] + a.c[i]) * dv;
        acc[2] += dv * a.Kd[i];
      }
      acc[3] += -(bl - bu) * dv;
      acc[5] += (hl ? log(gl) : 0.0) + (hu ? log(gu) : 0.0);
    } else {
      const double v = a.P[i] + a.alpha * a.dP[i];
      acc[1] += (hl ? log(v - l) : 0.0) + (hu ? log(u - v) : 0.0);
    }
  }
  for (int64_t j = t0; j < m; j += ts) {
    if (MODE == 0) {
      acc[1] = fmax(acc[1], fabs(a.res_p[j]));
    } else if (MODE == 1) {
      acc[0] -= 0.5 * a.y[j] * a.Kxy[d.n + j];
      acc[1] -= a.y[j] * a.Kd[d.n + j];
      acc[4] += fabs(a.res_p[j]);
    } else {
      const double dr = a.Kd[d.n + j] - (j >= d.m_E ? a.dP[d.n + j - d.m_E] : 0.0);
      acc[0] += fabs(a.res_p[j] + a.alpha * dr);
    }
  }
  __shared__ double sh[IT / 32][NOUT];
  __shared__ bool last;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 0; k < NV; k++) {
    const double v = wred(acc[k], IS_MAX[MODE][k]);
    if (lane == 0) sh[warp][k] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 0; k < NV; k++) {
      double v = sh[0][k];
      for (int w = 1; w < IT / 32; w++) v = IS_MAX[MODE][k] ? fmax(v, sh[w][k]) : v + sh[w][k];
      partials[(size_t)blockIdx.x * NOUT + k] = v;
    }
    __threadfence();
    last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last) {
    // the whole last CTA combines the per-CTA partials: thread t takes blocks t, t + IT, ...
    // in order, then the same fixed warp / CTA tree as above (deterministic)
    __threadfence();
    double v2[NV];
#pragma unroll
    for (int k = 0; k < NV; k++) v2[k] = 0.0;   // (the max-reduced values are absolute values)
    for (unsigned b = threadIdx.x; b < gridDim.x; b += IT)
#pragma unroll
      for (int k = 0; k < NV; k++) {
        const double w = __ldcg(&partials[(size_t)b * NOUT + k]);
        v2[k] = IS_MAX[MODE][k] ? fmax(v2[k], w) : v2[k] + w;
      }
    __syncthreads();   // (sh is reused)
#pragma unroll
    for (int k = 0; k < NV; k++) {
      const double v = wred(v2[k], IS_MAX[MODE][k]);
      if (lane == 0) sh[warp][k] = v;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int k = 0; k < NV; k++) {
        double v = sh[0][k];
        for (int w = 1; w < IT / 32; w++) v = IS_MAX[MODE][k] ? fmax(v, sh[w][k]) : v + sh[w][k];
        out[k] = v;
      }
      *counter = 0u;
    }
  }
}

// apply: P += a dP, y += a dy, z += a_d dz then the dual safeguard clip into
// [mu/(kS gap), kS mu/gap]; xy = (x, y) mirror for the next K0 product.
__global__ void __launch_bounds__(IT) k_ipm_apply(IpmDims d, double* __restrict__ P, double* __restrict__ zl,
                                                  double* __restrict__ zu, double* __restrict__ y,
                                                  double* __restrict__ xy, const double* __restrict__ dP,
                                                  const double* __restrict__ dzl, const double* __restrict__ dzu,
                                                  const double* __restrict__ dy, const double* __restrict__ lo,
                                                  const double* __restrict__ up, double alpha, double alpha_d,
                                                  double mu, double kappa_sigma) {
  pdl_wait();
  pdl_trigger();
  const int64_t np = d.n + d.m_I, m = d.m_E + d.m_I;
  for (int64_t i = blockIdx.x * (int64_t)IT + threadIdx.x; i < np; i += (int64_t)gridDim.x * IT) {
    const double v = P[i] + alpha * dP[i];
    P[i] = v;
    if (i < d.n) xy[i] = v;
    const double l = lo[i], u = up[i];
    if (fin(l)) {
      const double g = v - l, z = zl[i] + alpha_d * dzl[i];
      zl[i] = fmin(fmax(z, mu / (kappa_sigma * g)), kappa_sigma * mu / g);
    }
    if (fin(u)) {
      const double g = u - v, z = zu[i] + alpha_d * dzu[i];
      zu[i] = fmin(fmax(z, mu / (kappa_sigma * g)), kappa_sigma * mu / g);
    }
  }
  for (int64_t j = blockIdx.x * (int64_t)IT + threadIdx.x; j < m; j += (int64_t)gridDim.x * IT) {
    const double v = y[j] + alpha * dy[j];
    y[j] = v;
    xy[d.n + j] = v;
  }
}

int ipm_grid(int64_t n) { return (int)std::min<int64_t>(std::max<int64_t>(mds_cdiv(n, IT * 4), 1), 148 * 4); }
}  // namespace

extern "C" size_t ipm_workspace_size(int64_t n, int64_t m_I) {
  return 256 + sizeof(double) * NOUT * (size_t)ipm_grid(n + m_I);
}

extern "C" int ipm_rhs(int64_t n, int64_t m_E, int64_t m_I, const double* Kxy, const double* c, const double* g_E,
                       const double* P, const double* lo, const double* up, const double* zl, const double* zu,
                       const double* y, double mu, double* sigma, double* r, double* q, double* res_d, double* res_p,
                       void* stream) {
  if (n < 0 || m_E < 0 || m_I < 0 || !(mu >= 0.0)) return MDS_ERR_ARG;
  if (!Kxy || !c || !P || !lo || !up || !zl || !zu || !sigma || !r || !res_d || (m_E > 0 && !g_E) ||
      (m_E + m_I > 0 && (!y || !res_p)) || (m_I > 0 && !q))
    return MDS_ERR_ARG;
  const IpmDims d = {n, m_E, m_I};
  cudaStream_t st = (cudaStream_t)stream;
  MDS_LAUNCH(PC_VECTORS, st, MDS_CUDA_TRY(launch_pdl(k_ipm_rhs, dim3(ipm_grid(n + m_I)), dim3(IT), 0, st, d, Kxy, c,
                                                     g_E, P, lo, up, zl, zu, y, mu, sigma, r, q, res_d, res_p)));
  return MDS_OK;
}

extern "C" int ipm_directions(int64_t n, int64_t m_E, int64_t m_I, const double* dxy, const double* q,
                              const double* sigma, const double* P, const double* lo, const double* up,
                              const double* zl, const double* zu, double mu, double* dP, double* dzl, double* dzu,
                              double* dx0, void* stream) {
  if (n < 0 || m_E < 0 || m_I < 0) return MDS_ERR_ARG;
  if (!dxy || !sigma || !P || !lo || !up || !zl || !zu || !dP || !dzl || !dzu || !dx0 || (m_I > 0 && !q))
    return MDS_ERR_ARG;
  const IpmDims d = {n, m_E, m_I};
  cudaStream_t st = (cudaStream_t)stream;
  MDS_LAUNCH(PC_VECTORS, st, MDS_CUDA_TRY(launch_pdl(k_ipm_dir, dim3(ipm_grid(n + m_I)), dim3(IT), 0, st, d, dxy, q,
                                                     sigma, P, lo, up, zl, zu, mu, dP, dzl, dzu, dx0)));
  return MDS_OK;
}

extern "C" int ipm_reduce(int mode, int64_t n, int64_t m_E, int64_t m_I, const double* P, const double* dP,
                          const double* lo, const double* up, const double* zl, const double* zu, const double* y,
                          const double* c, const double* Kxy, const double* Kd, const double* res_d,
                          const double* res_p, double mu, double alpha, double* out, void* work, size_t work_bytes,
                          void* stream) {
  if (n < 0 || m_E < 0 || m_I < 0 || mode < 0 || mode > 2 || !out || !P || !lo || !up) return MDS_ERR_ARG;
  if (mode == 0 && (!zl || !zu || !res_d || (m_E + m_I > 0 && !res_p))) return MDS_ERR_ARG;
  if (mode == 1 && (!dP || !c || !Kxy || !Kd || (m_E + m_I > 0 && (!y || !res_p)))) return MDS_ERR_ARG;
  if (mode == 2 && (!dP || (m_E + m_I > 0 && (!Kd || !res_p)))) return MDS_ERR_ARG;
  if (!work || work_bytes < ipm_workspace_size(n, m_I)) return MDS_ERR_WORKSPACE;
  const IpmDims d = {n, m_E, m_I};
  RedIn a = {P, dP, lo, up, zl, zu, y, c, Kxy, Kd, res_d, res_p, mu, alpha};
  unsigned* counter = reinterpret_cast<unsigned*>(work);
  double* partials = reinterpret_cast<double*>(reinterpret_cast<char*>(work) + 256);
  cudaStream_t st = (cudaStream_t)stream;
  const dim3 g(ipm_grid(n + m_I));
  if (mode == 0)
    MDS_LAUNCH(PC_VECTORS, st, MDS_CUDA_TRY(launch_pdl(k_ipm_reduce<0>, g, dim3(IT), 0, st, d, a, partials, counter, out)));
  else if (mode == 1)
    MDS_LAUNCH(PC_VECTORS, st, MDS_CUDA_TRY(launch_pdl(k_ipm_reduce<1>, g, dim3(IT), 0, st, d, a, partials, counter, out)));
  else
    MDS_LAUNCH(PC_VECTORS, st, MDS_CUDA_TRY(launch_pdl(k_ipm_reduce<2>, g, dim3(IT), 0, st, d, a, partials, counter, out)));
  return MDS_OK;
}

extern "C" int ipm_apply(int64_t n, int64_t m_E, int64_t m_I, double* P, double* zl, double* zu, double* y, double* xy,
                         const double* dP, const double* dzl, const double* dzu, const double* dy, const double* lo,
                         const double* up, double alpha, double alpha_d, double mu, double kappa_sigma, void* stream) {
  if (n < 0 || m_E < 0 || m_I < 0 || !P || !zl || !zu || !xy || !dP || !dzl || !dzu || !lo || !up ||
      (m_E + m_I > 0 && (!y || !dy)) || !(kappa_sigma >= 1.0))
    return MDS_ERR_ARG;
  const IpmDims d = {n, m_E, m_I};
  cudaStream_t st = (cudaStream_t)stream;
  MDS_LAUNCH(PC_VECTORS, st, MDS_CUDA_TRY(launch_pdl(k_ipm_apply, dim3(ipm_grid(n + m_I)), dim3(IT), 0, st, d, P, zl,
                                                     zu, y, xy, dP, dzl, dzu, dy, lo, up, alpha, alpha_d, mu,
                                                     kappa_sigma)));
  return MDS_OK;
}
