// solve.cu — mds_solve: x = P^T L^{-T} D^{-1} L^{-1} P rhs_c with mds_factor's
// explicit-permutation factors (K4 solve), then the sparse
// step recovery dx_s = w .* (r_xs - J_s dy) (K2; first block row
// of Eq.(5)).  HBM-bound: L is streamed once per triangular sweep.
//
// Triangular sweeps are single "sync-free" launches: CTA i (row block of 64,
// index taken from an atomic ticket so lower blocks always run first) streams
// its part of L against already-published blocks (per-block ready flags), then
// solves its 64x64 diagonal block in one warp and publishes.
#include <algorithm>

#include "common.cuh"

const int32_t* mds_plan_rowptr(const mds_plan* P);
const int32_t* mds_plan_colidx(const mds_plan* P);
double* mds_factor_tol_ptr(const void* fwork);

namespace {
constexpr int TB = 64;        // row block
constexpr int ST = 256;       // threads
constexpr int PERM_MASK = (1 << 29) - 1;

struct SWork {
  double* y;
  int* flags;     // [nblk]
  int* tickets;   // [2]
};

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }
SWork carve(void* work, int64_t N, size_t* total) {
  SWork s;
  size_t off = 0;
  char* b = reinterpret_cast<char*>(work);
  auto take = [&](size_t bytes) { char* p = b + off; off = align_up(off + bytes, 256); return p; };
  s.tickets = reinterpret_cast<int*>(take(sizeof(int) * 4));
  s.flags = reinterpret_cast<int*>(take(sizeof(int) * (N / TB + 2)));
  s.y = reinterpret_cast<double*>(take(sizeof(double) * std::max<int64_t>(N, 1)));
  if (total) *total = off;
  return s;
}

__device__ __forceinline__ double ld_cg(const double* p) { return __ldcg(p); }

__global__ void k_gather(int64_t N, const int32_t* __restrict__ piv, const double* __restrict__ b,
                         double* __restrict__ y) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = b[piv[N + i] & PERM_MASK];
}

// forward: L y = y (unit lower; 2x2 D off-diagonals were moved out of L by the factor)
__global__ void __launch_bounds__(ST) k_trsv_fwd(int64_t N, const double* __restrict__ L, int64_t lda, double* y,
                                                 int* flags, int* ticket) {
  __shared__ int s_i;
  __shared__ double part[ST / TB][TB];
  __shared__ double Ld[TB * (TB + 1)];
  if (threadIdx.x == 0) s_i = atomicAdd(ticket, 1);
  __syncthreads();
  const int64_t i = s_i;
  const int64_t r0 = i * TB;
  const int nr = (int)((N - r0) < TB ? (N - r0) : TB);
  const int r = threadIdx.x & (TB - 1), cgp = threadIdx.x / TB;   // 4 column groups of 16
  // stage the diagonal block while waiting
  for (int idx = threadIdx.x; idx < TB * TB; idx += ST) {
    const int rr = idx % TB, cc = idx / TB;
    Ld[cc * (TB + 1) + rr] = (rr < nr && cc < nr && rr > cc) ? L[(r0 + rr) + (r0 + cc) * lda] : 0.0;
  }
  double acc = 0.0;
  for (int64_t q = 0; q < i; q++) {
    if (threadIdx.x == 0) {
      while (atomicAdd(&flags[q], 0) == 0) { __nanosleep(32); }
    }
    __syncthreads();
    const int64_t c0 = q * TB + cgp * 16;
    if (r < nr) {
#pragma unroll
      for (int c = 0; c < 16; c++) acc += L[(r0 + r) + (c0 + c) * lda] * ld_cg(&y[c0 + c]);
    }
  }
  part[cgp][r] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    double v0 = 0.0, v1 = 0.0;
    if (lane < nr) v0 = ld_cg(&y[r0 + lane]) - (part[0][lane] + part[1][lane] + part[2][lane] + part[3][lane]);
    if (lane + 32 < nr)
      v1 = ld_cg(&y[r0 + lane + 32]) -
           (part[0][lane + 32] + part[1][lane + 32] + part[2][lane + 32] + part[3][lane + 32]);
    for (int c = 0; c < nr; c++) {
      const double yc = __shfl_sync(0xffffffffu, c < 32 ? v0 : v1, c & 31);
      if (lane > c) v0 -= Ld[c * (TB + 1) + lane] * yc;
      if (lane + 32 > c) v1 -= Ld[c * (TB + 1) + lane + 32] * yc;
    }
    if (lane < nr) y[r0 + lane] = v0;
    if (lane + 32 < nr) y[r0 + lane + 32] = v1;
    __threadfence();
    __syncwarp();
    if (lane == 0) atomicExch(&flags[i], 1);
  }
}

// D solve: 1x1 and 2x2 blocks (LAPACK dsytrs scaled 2x2 formula); 2x2 off-diagonal at (k, k+1) (upper slot)
__global__ void k_dsolve(int64_t N, const double* __restrict__ LD, int64_t lda, const int32_t* __restrict__ piv,
                         double* y, const double* tolp, double tolv, int32_t* status) {
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

// backward: L^T x = z, blocks from the bottom
__global__ void __launch_bounds__(ST) k_trsv_bwd(int64_t N, const double* __restrict__ L, int64_t lda, double* y,
                                                 int* flags, int* ticket) {
  __shared__ int s_i;
  __shared__ double Ld[TB * (TB + 1)];
  __shared__ double colsum[TB];
  const int64_t nblk = (N + TB - 1) / TB;
  if (threadIdx.x == 0) s_i = atomicAdd(ticket, 1);
  __syncthreads();
  const int64_t i = nblk - 1 - s_i;
  const int64_t r0 = i * TB;
  const int nr = (int)((N - r0) < TB ? (N - r0) : TB);
  for (int idx = threadIdx.x; idx < TB * TB; idx += ST) {
    const int rr = idx % TB, cc = idx / TB;
    Ld[cc * (TB + 1) + rr] = (rr < nr && cc < nr && rr > cc) ? L[(r0 + rr) + (r0 + cc) * lda] : 0.0;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // warp w owns columns c = w + 8*u (u < 8) of this block; lanes stride rows of later blocks
  double acc[8];
#pragma unroll
  for (int u = 0; u < 8; u++) acc[u] = 0.0;
  for (int64_t q = nblk - 1; q > i; q--) {   // completion order: last block finishes first
    if (threadIdx.x == 0) {
      while (atomicAdd(&flags[q], 0) == 0) { __nanosleep(32); }
    }
    __syncthreads();
    const int64_t q0 = q * TB;
    const int qn = (int)((N - q0) < TB ? (N - q0) : TB);
    const double x0 = (lane < qn) ? ld_cg(&y[q0 + lane]) : 0.0;
    const double x1 = (lane + 32 < qn) ? ld_cg(&y[q0 + lane + 32]) : 0.0;
#pragma unroll
    for (int u = 0; u < 8; u++) {
      const int c = warp + 8 * u;
      if (c < nr) {
        const double* Lc = L + (r0 + c) * lda + q0;
        double s = 0.0;
        if (lane < qn) s += Lc[lane] * x0;
        if (lane + 32 < qn) s += Lc[lane + 32] * x1;
        acc[u] += s;
      }
    }
  }
#pragma unroll
  for (int u = 0; u < 8; u++) {
    const double v = warp_sum(acc[u]);
    if (lane == 0) colsum[warp + 8 * u] = v;
  }
  __syncthreads();
  if (warp == 0) {
    double v0 = 0.0, v1 = 0.0;
    if (lane < nr) v0 = ld_cg(&y[r0 + lane]) - colsum[lane];
    if (lane + 32 < nr) v1 = ld_cg(&y[r0 + lane + 32]) - colsum[lane + 32];
    for (int c = nr - 1; c >= 0; c--) {
      const double xc = __shfl_sync(0xffffffffu, c < 32 ? v0 : v1, c & 31);
      // row c of L (columns < c) : v_{c'} -= L[c, c'] * x_c
      if (lane < c) v0 -= Ld[lane * (TB + 1) + c] * xc;
      if (lane + 32 < c) v1 -= Ld[(lane + 32) * (TB + 1) + c] * xc;
    }
    if (lane < nr) y[r0 + lane] = v0;
    if (lane + 32 < nr) y[r0 + lane + 32] = v1;
    __threadfence();
    __syncwarp();
    if (lane == 0) atomicExch(&flags[i], 1);
  }
}

__global__ void k_scatter(int64_t N, const int32_t* __restrict__ piv, const double* __restrict__ y,
                          double* __restrict__ x) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
    x[piv[N + i] & PERM_MASK] = y[i];
}

// dx_s[k] = w[k] * (r_xs[k] - sum_p val[p] * dy[colidx[p]])
__global__ void k_recover(int64_t n_s, const int32_t* __restrict__ rowptr, const int32_t* __restrict__ colidx,
                          const double* __restrict__ val, const double* __restrict__ w,
                          const double* __restrict__ r_xs, const double* __restrict__ dy,
                          double* __restrict__ dx_s) {
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

extern "C" int mds_solve(const mds_plan* plan, int64_t N, const double* LD, int64_t ldm, const int32_t* piv,
                         const double* rhs_c, const double* js_val, const double* w, const double* r_xs,
                         double* dxy, double* dx_s, double zero_tol, const void* fwork, int32_t* status,
                         void* work, size_t work_bytes, void* stream) {
  if (N < 0 || (N > 0 && (!LD || !piv || !rhs_c || !dxy)) || ldm < std::max<int64_t>(N, 1)) return MDS_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  if (!work || work_bytes < mds_solve_workspace_size(N)) return MDS_ERR_WORKSPACE;
  if (N > 0) {
    SWork s = carve(work, N, nullptr);
    const int64_t nblk = (N + TB - 1) / TB;
    MDS_CUDA_TRY(cudaMemsetAsync(s.tickets, 0, sizeof(int) * 4, st));
    MDS_CUDA_TRY(cudaMemsetAsync(s.flags, 0, sizeof(int) * (nblk + 1), st));
    const unsigned ge = (unsigned)std::min<int64_t>(mds_cdiv(N, 256), 148 * 8);
    MDS_LAUNCH(PC_SOLVE_GATHER, st, (k_gather<<<ge, 256, 0, st>>>(N, piv, rhs_c, s.y)));
    MDS_LAUNCH(PC_SOLVE_FWD, st, (k_trsv_fwd<<<(unsigned)nblk, ST, 0, st>>>(N, LD, ldm, s.y, s.flags, s.tickets)));
    const double* tolp = (zero_tol < 0.0 && fwork) ? mds_factor_tol_ptr(fwork) : nullptr;
    MDS_LAUNCH(PC_SOLVE_D, st,
               (k_dsolve<<<ge, 256, 0, st>>>(N, LD, ldm, piv, s.y, tolp, zero_tol < 0.0 ? 0.0 : zero_tol, status)));
    MDS_CUDA_TRY(cudaMemsetAsync(s.flags, 0, sizeof(int) * (nblk + 1), st));
    MDS_LAUNCH(PC_SOLVE_BWD, st,
               (k_trsv_bwd<<<(unsigned)nblk, ST, 0, st>>>(N, LD, ldm, s.y, s.flags, s.tickets + 1)));
    MDS_LAUNCH(PC_SOLVE_SCATTER, st, (k_scatter<<<ge, 256, 0, st>>>(N, piv, s.y, dxy)));
  }
  if (plan && dx_s) {
    int64_t dims[5];
    mds_plan_dims(plan, dims);
    const int64_t n_s = dims[0], n_d = dims[1];
    if (dims[1] + dims[2] + dims[3] != N) return MDS_ERR_ARG;
    if (n_s > 0) {
      if (!w || !r_xs || (dims[4] > 0 && !js_val)) return MDS_ERR_ARG;
      const unsigned g = (unsigned)std::min<int64_t>(mds_cdiv(n_s, 256), 148 * 16);
      MDS_LAUNCH(PC_RECOVER, st,
                 (k_recover<<<g, 256, 0, st>>>(n_s, mds_plan_rowptr(plan), mds_plan_colidx(plan), js_val, w, r_xs,
                                               dxy + n_d, dx_s)));
    }
  }
  return MDS_OK;
}
