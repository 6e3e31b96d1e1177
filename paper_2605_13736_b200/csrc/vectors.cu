// vectors.cu — ipm_step_vectors: the barrier vector kernels (K1)
// in ONE fused HBM pass: fraction-to-boundary min-reductions,
// complementarity max/sum, residual inf-norms, optional barrier diagonal sigma.
// Grid-stride over n with 128-bit loads; per-CTA partials reduced by the last
// CTA to finish (deterministic fixed-order final reduction).  Bytes/element:
// 8 inputs x 8 B (+8 B sigma write) — HBM-bound.
#include <algorithm>

#include "common.cuh"

namespace {
constexpr int VT = 256;             // threads per CTA
constexpr int MAXRES = 8;
constexpr int NPART = 6 + MAXRES;   // partial slots per CTA

struct ResPtrs {
  const double* p[MAXRES];
  int64_t len[MAXRES];
  int64_t str[MAXRES];   // batched: per-scenario element stride of residual j
  int n;
};
// batched (ipm_step_vectors_batched): scenario s = blockIdx.y reads the 8 vectors and
// writes sigma at + s * vec, out at + s * out, status + s, its own partials / counter
struct VStr {
  int64_t vec, out;
  const double* tau_arr;   // [batch] or NULL (scalar tau)
  const double* mu_arr;    // [batch] or NULL (scalar mu)
  int batched;
};

struct Part {
  double ap, ad, cinf, csum, nc;
  long long bad;
  double res[MAXRES];
};

__device__ __forceinline__ void elem(int64_t i, double x, double dx, double lo, double up, double zl, double zu,
                                     double dzl, double dzu, double tau, double mu, Part& P, double* sigma) {
  const bool hl = fabs(lo) < MDS_INF_BOUND, hu = fabs(up) < MDS_INF_BOUND;
  double s = 0.0;
  if (hl) {
    const double gap = __dsub_rn(x, lo);
    if (!(gap > 0.0) || !(zl > 0.0)) P.bad = min(P.bad, (long long)i);
    if (dx < 0.0) P.ap = fmin(P.ap, __ddiv_rn(__dmul_rn(tau, gap), -dx));
    if (dzl < 0.0) P.ad = fmin(P.ad, __ddiv_rn(__dmul_rn(tau, zl), -dzl));
    const double c = __dmul_rn(gap, zl);
    P.cinf = fmax(P.cinf, fabs(__dsub_rn(c, mu)));
    P.csum += c;
    P.nc += 1.0;
    s = __dadd_rn(s, __ddiv_rn(zl, gap));
  }
  if (hu) {
    const double gap = __dsub_rn(up, x);
    if (!(gap > 0.0) || !(zu > 0.0)) P.bad = min(P.bad, (long long)i);
    if (dx > 0.0) P.ap = fmin(P.ap, __ddiv_rn(__dmul_rn(tau, gap), dx));
    if (dzu < 0.0) P.ad = fmin(P.ad, __ddiv_rn(__dmul_rn(tau, zu), -dzu));
    const double c = __dmul_rn(gap, zu);
    P.cinf = fmax(P.cinf, fabs(__dsub_rn(c, mu)));
    P.csum += c;
    P.nc += 1.0;
    s = __dadd_rn(s, __ddiv_rn(zu, gap));
  }
  if (sigma) sigma[i] = s;
}

__global__ void __launch_bounds__(VT)
k_step_vectors(int64_t n, const double* __restrict__ x, const double* __restrict__ dx,
               const double* __restrict__ lo, const double* __restrict__ up,
               const double* __restrict__ zl, const double* __restrict__ zu,
               const double* __restrict__ dzl, const double* __restrict__ dzu,
               double tau, double mu, ResPtrs R, double* __restrict__ out, double* __restrict__ sigma,
               int32_t* status, double* __restrict__ partials, unsigned int* counter, VStr z) {
  pdl_wait();
  pdl_trigger();
  if (z.batched) {
    const int64_t s = blockIdx.y, o = s * z.vec;
    x += o; dx += o; lo += o; up += o; zl += o; zu += o; dzl += o; dzu += o;
    if (sigma) sigma += o;
    out += s * z.out;
    if (status) status += s;
    partials += s * (int64_t)gridDim.x * NPART;
    counter += s;
    if (z.tau_arr) tau = z.tau_arr[s];
    if (z.mu_arr) mu = z.mu_arr[s];
    for (int j = 0; j < R.n; j++) R.p[j] += s * R.str[j];
  }
  Part P;
  P.ap = 1.0; P.ad = 1.0; P.cinf = 0.0; P.csum = 0.0; P.nc = 0.0; P.bad = LLONG_MAX;
#pragma unroll
  for (int j = 0; j < MAXRES; j++) P.res[j] = 0.0;
  const int64_t tid = blockIdx.x * (int64_t)VT + threadIdx.x;
  const int64_t nthr = (int64_t)gridDim.x * VT;
  // pairs of elements with 128-bit loads when all arrays are 16-byte aligned
  const bool al = ((((uintptr_t)x | (uintptr_t)dx | (uintptr_t)lo | (uintptr_t)up | (uintptr_t)zl | (uintptr_t)zu |
                     (uintptr_t)dzl | (uintptr_t)dzu | (uintptr_t)sigma) & 15) == 0);
  if (al) {
    const int64_t n2 = n / 2;
    for (int64_t t = tid; t < n2; t += nthr) {
      double2 X = reinterpret_cast<const double2*>(x)[t], DX = reinterpret_cast<const double2*>(dx)[t];
      double2 LO = reinterpret_cast<const double2*>(lo)[t], UP = reinterpret_cast<const double2*>(up)[t];
      double2 ZL = reinterpret_cast<const double2*>(zl)[t], ZU = reinterpret_cast<const double2*>(zu)[t];
      double2 DZL = reinterpret_cast<const double2*>(dzl)[t], DZU = reinterpret_cast<const double2*>(dzu)[t];
      elem(2 * t, X.x, DX.x, LO.x, UP.x, ZL.x, ZU.x, DZL.x, DZU.x, tau, mu, P, sigma);
      elem(2 * t + 1, X.y, DX.y, LO.y, UP.y, ZL.y, ZU.y, DZL.y, DZU.y, tau, mu, P, sigma);
    }
    if (tid == 0 && (n & 1)) {
      int64_t i = n - 1;
      elem(i, x[i], dx[i], lo[i], up[i], zl[i], zu[i], dzl[i], dzu[i], tau, mu, P, sigma);
    }
  } else {
    for (int64_t i = tid; i < n; i += nthr)
      elem(i, x[i], dx[i], lo[i], up[i], zl[i], zu[i], dzl[i], dzu[i], tau, mu, P, sigma);
  }
  for (int j = 0; j < R.n; j++) {
    const double* v = R.p[j];
    double mx = 0.0;
    if ((((uintptr_t)v) & 15) == 0) {
      const int64_t h = R.len[j] / 2;
      for (int64_t t = tid; t < h; t += nthr) {
        const double2 q = reinterpret_cast<const double2*>(v)[t];
        mx = fmax(mx, fmax(fabs(q.x), fabs(q.y)));
      }
      if (tid == 0 && (R.len[j] & 1)) mx = fmax(mx, fabs(v[R.len[j] - 1]));
    } else {
      for (int64_t i = tid; i < R.len[j]; i += nthr) mx = fmax(mx, fabs(v[i]));
    }
    P.res[j] = mx;
  }
  // CTA reduction (fixed order)
  __shared__ double sh[VT / 32][NPART];
  __shared__ long long shb[VT / 32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double a0 = warp_min(P.ap), a1 = warp_min(P.ad), a2 = warp_max(P.cinf), a3 = warp_sum(P.csum), a4 = warp_sum(P.nc);
  long long b = P.bad;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) b = min(b, (long long)__shfl_xor_sync(0xffffffffu, b, o));
  double rr[MAXRES];
#pragma unroll
  for (int j = 0; j < MAXRES; j++) rr[j] = warp_max(P.res[j]);
  if (lane == 0) {
    sh[warp][0] = a0; sh[warp][1] = a1; sh[warp][2] = a2; sh[warp][3] = a3; sh[warp][4] = a4;
    shb[warp] = b;
#pragma unroll
    for (int j = 0; j < MAXRES; j++) sh[warp][6 + j] = rr[j];
  }
  __syncthreads();
  __shared__ bool last;
  if (threadIdx.x == 0) {
    double q0 = sh[0][0], q1 = sh[0][1], q2 = sh[0][2], q3 = sh[0][3], q4 = sh[0][4];
    long long qb = shb[0];
    double qr[MAXRES];
    for (int j = 0; j < MAXRES; j++) qr[j] = sh[0][6 + j];
    for (int w = 1; w < VT / 32; w++) {
      q0 = fmin(q0, sh[w][0]); q1 = fmin(q1, sh[w][1]); q2 = fmax(q2, sh[w][2]);
      q3 += sh[w][3]; q4 += sh[w][4]; qb = min(qb, shb[w]);
      for (int j = 0; j < MAXRES; j++) qr[j] = fmax(qr[j], sh[w][6 + j]);
    }
    double* my = partials + (size_t)blockIdx.x * NPART;
    my[0] = q0; my[1] = q1; my[2] = q2; my[3] = q3; my[4] = q4;
    my[5] = __longlong_as_double(qb);
    for (int j = 0; j < MAXRES; j++) my[6 + j] = qr[j];
    __threadfence();
    unsigned prev = atomicAdd(counter, 1u);
    last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return;
  // last CTA: fixed-order tree reduction over the CTA partials (deterministic: the
  // assignment of partials to threads and the combining tree depend only on the grid)
  __threadfence();
  {
    double q0 = 1.0, q1 = 1.0, q2 = 0.0, q3 = 0.0, q4 = 0.0;
    long long qb = LLONG_MAX;
    double qr[MAXRES];
#pragma unroll
    for (int j = 0; j < MAXRES; j++) qr[j] = 0.0;
    for (unsigned c = threadIdx.x; c < gridDim.x; c += VT) {
      const double* my = partials + (size_t)c * NPART;
      q0 = fmin(q0, __ldcg(my + 0)); q1 = fmin(q1, __ldcg(my + 1)); q2 = fmax(q2, __ldcg(my + 2));
      q3 += __ldcg(my + 3); q4 += __ldcg(my + 4);
      qb = min(qb, __double_as_longlong(__ldcg(my + 5)));
#pragma unroll
      for (int j = 0; j < MAXRES; j++) qr[j] = fmax(qr[j], __ldcg(my + 6 + j));
    }
    q0 = warp_min(q0); q1 = warp_min(q1); q2 = warp_max(q2); q3 = warp_sum(q3); q4 = warp_sum(q4);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) qb = min(qb, (long long)__shfl_xor_sync(0xffffffffu, qb, o));
#pragma unroll
    for (int j = 0; j < MAXRES; j++) qr[j] = warp_max(qr[j]);
    __syncthreads();
    if (lane == 0) {
      sh[warp][0] = q0; sh[warp][1] = q1; sh[warp][2] = q2; sh[warp][3] = q3; sh[warp][4] = q4;
      shb[warp] = qb;
#pragma unroll
      for (int j = 0; j < MAXRES; j++) sh[warp][6 + j] = qr[j];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double r0 = sh[0][0], r1 = sh[0][1], r2 = sh[0][2], r3 = sh[0][3], r4 = sh[0][4];
      long long rb = shb[0];
      double rr2[MAXRES];
      for (int j = 0; j < MAXRES; j++) rr2[j] = sh[0][6 + j];
      for (int w = 1; w < VT / 32; w++) {
        r0 = fmin(r0, sh[w][0]); r1 = fmin(r1, sh[w][1]); r2 = fmax(r2, sh[w][2]);
        r3 += sh[w][3]; r4 += sh[w][4]; rb = min(rb, shb[w]);
        for (int j = 0; j < MAXRES; j++) rr2[j] = fmax(rr2[j], sh[w][6 + j]);
      }
      out[0] = r0; out[1] = r1; out[2] = r2; out[3] = r3; out[4] = r4;
      out[5] = (rb == LLONG_MAX) ? -1.0 : (double)rb;
      for (int j = 0; j < R.n; j++) out[6 + j] = rr2[j];
      if (rb != LLONG_MAX) mds_set_status(status, MDS_ERR_NOT_INTERIOR);
      *counter = 0u;   // leave the workspace reusable (graph replays)
    }
  }
}

int vec_grid(int64_t n) {
  int64_t b = mds_cdiv(std::max<int64_t>(n, 1), 2 * VT * 4);
  return (int)std::min<int64_t>(std::max<int64_t>(b, 1), 148 * 8);
}
}  // namespace

extern "C" size_t ipm_step_vectors_workspace_size(int64_t n) {
  return 256 + sizeof(double) * NPART * (size_t)vec_grid(n);
}

extern "C" int ipm_step_vectors(int64_t n, const double* x, const double* dx, const double* lo, const double* up,
                                const double* zl, const double* zu, const double* dzl, const double* dzu,
                                double tau, double mu, int32_t n_res, const double* const* res,
                                const int64_t* res_len, double* out, double* sigma_out, int32_t* status,
                                void* work, size_t work_bytes, void* stream) {
  if (n < 0 || !out || n_res < 0 || n_res > MAXRES) return MDS_ERR_ARG;
  if (n > 0 && (!x || !dx || !lo || !up || !zl || !zu || !dzl || !dzu)) return MDS_ERR_ARG;
  if (n_res > 0 && (!res || !res_len)) return MDS_ERR_ARG;
  if (!work || work_bytes < ipm_step_vectors_workspace_size(n)) return MDS_ERR_WORKSPACE;
  ResPtrs R;
  R.n = n_res;
  for (int j = 0; j < MAXRES; j++) { R.p[j] = nullptr; R.len[j] = 0; R.str[j] = 0; }
  for (int j = 0; j < n_res; j++) {
    if (res_len[j] < 0 || (res_len[j] > 0 && !res[j])) return MDS_ERR_ARG;
    R.p[j] = res[j]; R.len[j] = res_len[j];
  }
  unsigned int* counter = reinterpret_cast<unsigned int*>(work);
  double* partials = reinterpret_cast<double*>(reinterpret_cast<char*>(work) + 256);
  int grid = vec_grid(n);
  cudaStream_t st = (cudaStream_t)stream;
  const VStr z = {};
  MDS_LAUNCH(PC_VECTORS, st,
             MDS_CUDA_TRY(launch_pdl(k_step_vectors, dim3(grid), dim3(VT), 0, st, n, x, dx, lo, up, zl, zu, dzl, dzu, tau,
                                     mu, R, out, sigma_out, status, partials, counter, z)));
  return MDS_OK;
}

static int vec_grid_b(int64_t n) { return std::min(vec_grid(n), 64); }

extern "C" size_t ipm_step_vectors_batched_workspace_size(int64_t n, int64_t batch) {
  if (batch < 1) return 0;
  return ((256 + 4 * (size_t)batch + 255) / 256) * 256 + sizeof(double) * NPART * (size_t)vec_grid_b(n) * batch;
}

// `batch` scenarios, each with n components at + s * str_vec (x, dx, lo, up, zl, zu, dzl,
// dzu, sigma_out), results at out + s * str_out, status[s]; tau / mu per scenario
// (tau_arr / mu_arr, device) or the scalars; residual j of scenario s at res[j] + s * res_str[j].
extern "C" int ipm_step_vectors_batched(int64_t batch, int64_t n, int64_t str_vec, const double* x, const double* dx,
                                        const double* lo, const double* up, const double* zl, const double* zu,
                                        const double* dzl, const double* dzu, double tau, double mu,
                                        const double* tau_arr, const double* mu_arr, int32_t n_res,
                                        const double* const* res, const int64_t* res_len, const int64_t* res_str,
                                        double* out, int64_t str_out, double* sigma_out, int32_t* status,
                                        void* work, size_t work_bytes, void* stream) {
  if (batch < 0 || n < 0 || n_res < 0 || n_res > MAXRES) return MDS_ERR_ARG;
  if (batch == 0) return MDS_OK;
  if (!out || !status || str_out < 6 + n_res || (n > 0 && str_vec < n)) return MDS_ERR_ARG;
  if (n > 0 && (!x || !dx || !lo || !up || !zl || !zu || !dzl || !dzu)) return MDS_ERR_ARG;
  if (n_res > 0 && (!res || !res_len || !res_str)) return MDS_ERR_ARG;
  if (!work || work_bytes < ipm_step_vectors_batched_workspace_size(n, batch)) return MDS_ERR_WORKSPACE;
  ResPtrs R;
  R.n = n_res;
  for (int j = 0; j < MAXRES; j++) { R.p[j] = nullptr; R.len[j] = 0; R.str[j] = 0; }
  for (int j = 0; j < n_res; j++) {
    if (res_len[j] < 0 || (res_len[j] > 0 && !res[j])) return MDS_ERR_ARG;
    R.p[j] = res[j]; R.len[j] = res_len[j]; R.str[j] = res_str[j];
  }
  unsigned int* counter = reinterpret_cast<unsigned int*>(work);
  double* partials = reinterpret_cast<double*>(reinterpret_cast<char*>(work) + ((256 + 4 * (size_t)batch + 255) / 256) * 256);
  const int grid = vec_grid_b(n);
  cudaStream_t st = (cudaStream_t)stream;
  // counters start at 0 (each scenario's last CTA resets its own); zero them once per call
  MDS_CUDA_TRY(cudaMemsetAsync(counter, 0, 4 * (size_t)batch, st));
  VStr z;
  z.vec = str_vec; z.out = str_out; z.tau_arr = tau_arr; z.mu_arr = mu_arr; z.batched = 1;
  MDS_LAUNCH(PC_VECTORS, st,
             MDS_CUDA_TRY(launch_pdl(k_step_vectors, dim3(grid, (unsigned)batch), dim3(VT), 0, st, n, x, dx, lo, up, zl,
                                     zu, dzl, dzu, tau, mu, R, out, sigma_out, status, partials, counter, z)));
  return MDS_OK;
}
