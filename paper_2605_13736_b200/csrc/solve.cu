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
  double* binv;   // [nblk][TB*TB] inverses of the unit-lower diagonal blocks (column-major)
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
  s.binv = reinterpret_cast<double*>(take(sizeof(double) * TB * TB * (N / TB + 1)));
  if (total) *total = off;
  return s;
}

__device__ __forceinline__ double ld_cg(const double* p) { return __ldcg(p); }

__global__ void k_gather(int64_t N, const int32_t* __restrict__ piv, const double* __restrict__ b,
                         double* __restrict__ y) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = b[piv[N + i] & PERM_MASK];
}

// Inverses of the unit-lower TB x TB diagonal blocks of L (one CTA per block,
// row-by-row: Binv[r][c] = -sum_{k=c}^{r-1} L[r][k] Binv[k][c]).  With them the
// dependent chain of the triangular sweeps is two small GEMVs per block.
__global__ void __launch_bounds__(256) k_inv_blocks(int64_t N, const double* __restrict__ L, int64_t lda,
                                                    double* __restrict__ binv) {
  extern __shared__ double ism[];
  double* Ls = ism;                      // Ls[k*(TB+1) + r] = L[r][k]
  double* Bs = ism + TB * (TB + 1);      // Bs[c*(TB+1) + r] = Binv[r][c]
  const int64_t i = blockIdx.x;
  const int64_t r0 = i * TB;
  const int nr = (int)((N - r0) < TB ? (N - r0) : TB);
  for (int idx = threadIdx.x; idx < TB * TB; idx += blockDim.x) {
    const int r = idx % TB, c = idx / TB;
    Ls[c * (TB + 1) + r] = (r < nr && c < nr && r > c) ? L[(r0 + r) + (r0 + c) * lda] : 0.0;
    Bs[c * (TB + 1) + r] = (r == c) ? 1.0 : 0.0;
  }
  __syncthreads();
  // 4 threads per column c split the dot product; rows r sequential
  const int c = threadIdx.x >> 2, part = threadIdx.x & 3;
  for (int r = 1; r < nr; r++) {
    double sacc = 0.0;
    if (c < r) {
      for (int k = c + part; k < r; k += 4) sacc += Ls[k * (TB + 1) + r] * Bs[c * (TB + 1) + k];
    }
    sacc += __shfl_xor_sync(0xffffffffu, sacc, 1);
    sacc += __shfl_xor_sync(0xffffffffu, sacc, 2);
    if (c < r && part == 0) Bs[c * (TB + 1) + r] = -sacc;
    __syncthreads();
  }
  double* out = binv + (size_t)i * TB * TB;
  for (int idx = threadIdx.x; idx < TB * TB; idx += blockDim.x) {
    const int r = idx % TB, cc = idx / TB;
    out[idx] = Bs[cc * (TB + 1) + r];
  }
}

// forward: L y = y (unit lower; 2x2 D off-diagonals were moved out of L by the factor).
// CTA i (ticket order) streams its row block of L against the published y_q, the
// loads of L for block q+1 issued before waiting on block q's flag; then
// y_i = Binv_i (b_i - acc).
__global__ void __launch_bounds__(ST) k_trsv_fwd(int64_t N, const double* __restrict__ L, int64_t lda, double* y,
                                                 const double* __restrict__ binv, int* flags, int* ticket) {
  __shared__ int s_i;
  __shared__ double part[ST / TB][TB];
  __shared__ double v[TB];
  if (threadIdx.x == 0) s_i = atomicAdd(ticket, 1);
  __syncthreads();
  const int64_t i = s_i;
  const int64_t r0 = i * TB;
  const int nr = (int)((N - r0) < TB ? (N - r0) : TB);
  const int r = threadIdx.x & (TB - 1), cgp = threadIdx.x / TB;   // 4 column groups of 16
  double acc = 0.0;
  double lv[16], ln[16];
  const double* Lr = L + (r0 + r);
  auto loadL = [&](int64_t q, double* dst) {
    const int64_t c0 = q * TB + cgp * 16;
#pragma unroll
    for (int c = 0; c < 16; c++) dst[c] = (r < nr) ? Lr[(c0 + c) * lda] : 0.0;
  };
  if (i > 0) loadL(0, lv);
  for (int64_t q = 0; q < i; q++) {
    if (q + 1 < i) loadL(q + 1, ln);
    if (threadIdx.x == 0) {
      while (*((volatile int*)&flags[q]) == 0) { }
      __threadfence();
    }
    __syncthreads();
    const double* yq = y + q * TB + cgp * 16;
#pragma unroll
    for (int c = 0; c < 16; c++) acc += lv[c] * ld_cg(&yq[c]);
#pragma unroll
    for (int c = 0; c < 16; c++) lv[c] = ln[c];
  }
  part[cgp][r] = acc;
  __syncthreads();
  if (threadIdx.x < TB) {
    const int rr = threadIdx.x;
    v[rr] = (rr < nr) ? ld_cg(&y[r0 + rr]) - (part[0][rr] + part[1][rr] + part[2][rr] + part[3][rr]) : 0.0;
  }
  __syncthreads();
  // y_i = Binv v : thread (r, cgp) sums 16 columns, reduce over the 4 groups
  const double* B = binv + (size_t)i * TB * TB;
  double sacc = 0.0;
#pragma unroll
  for (int c = 0; c < 16; c++) {
    const int cc = cgp * 16 + c;
    sacc += B[r + cc * TB] * v[cc];
  }
  part[cgp][r] = sacc;
  __syncthreads();
  if (threadIdx.x < TB) {
    const int rr = threadIdx.x;
    if (rr < nr) y[r0 + rr] = part[0][rr] + part[1][rr] + part[2][rr] + part[3][rr];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicExch(&flags[i], 1);
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

// backward: L^T x = z, blocks from the bottom.  CTA i accumulates
// sum_{q>i} L[q rows, i cols]^T x_q (threads run down contiguous column
// segments: thread (k, cg) owns row k of every later block and 16 columns),
// then x_i = Binv_i^T (z_i - acc).
__global__ void __launch_bounds__(ST) k_trsv_bwd(int64_t N, const double* __restrict__ L, int64_t lda, double* y,
                                                 const double* __restrict__ binv, int* flags, int* ticket) {
  __shared__ int s_i;
  __shared__ double redt[TB][TB + 1];
  __shared__ double part4[4][TB];
  __shared__ double v[TB];
  const int64_t nblk = (N + TB - 1) / TB;
  if (threadIdx.x == 0) s_i = atomicAdd(ticket, 1);
  __syncthreads();
  const int64_t i = nblk - 1 - s_i;
  const int64_t r0 = i * TB;
  const int nr = (int)((N - r0) < TB ? (N - r0) : TB);
  const int k = threadIdx.x & (TB - 1), cgp = threadIdx.x / TB;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double acc[16];
#pragma unroll
  for (int c = 0; c < 16; c++) acc[c] = 0.0;
  double lv[16], ln[16];
  auto loadL = [&](int64_t q, double* dst) {
    const int64_t row = q * TB + k;
    const bool ok = row < N;
#pragma unroll
    for (int c = 0; c < 16; c++) {
      const int cc = cgp * 16 + c;
      dst[c] = (ok && cc < nr) ? L[row + (r0 + cc) * lda] : 0.0;
    }
  };
  if (nblk - 1 > i) loadL(nblk - 1, lv);
  for (int64_t q = nblk - 1; q > i; q--) {   // completion order: last block finishes first
    if (q - 1 > i) loadL(q - 1, ln);
    if (threadIdx.x == 0) {
      while (*((volatile int*)&flags[q]) == 0) { }
      __threadfence();
    }
    __syncthreads();
    const int64_t row = q * TB + k;
    const double xq = (row < N) ? ld_cg(&y[row]) : 0.0;
#pragma unroll
    for (int c = 0; c < 16; c++) acc[c] += lv[c] * xq;
#pragma unroll
    for (int c = 0; c < 16; c++) lv[c] = ln[c];
  }
  // reduce acc over the 64 rows k: transpose through shared memory (no shuffle chains)
#pragma unroll
  for (int c = 0; c < 16; c++) redt[k][cgp * 16 + c] = acc[c];
  __syncthreads();
  {
    const int c = threadIdx.x & (TB - 1), part = threadIdx.x / TB;   // 4 threads per column, 16 rows each
    double sacc = 0.0;
#pragma unroll
    for (int kk = 0; kk < 16; kk++) sacc += redt[part * 16 + kk][c];
    part4[part][c] = sacc;
  }
  __syncthreads();
  if (threadIdx.x < TB) {
    const int cc = threadIdx.x;
    const double sum = part4[0][cc] + part4[1][cc] + part4[2][cc] + part4[3][cc];
    v[cc] = (cc < nr) ? ld_cg(&y[r0 + cc]) - sum : 0.0;
  }
  __syncthreads();
  // x_i = Binv^T v : x[c] = sum_r Binv[r][c] v[r]; thread (c = k, group cgp) sums 16 rows
  const double* B = binv + (size_t)i * TB * TB;
  double sacc = 0.0;
#pragma unroll
  for (int rr = 0; rr < 16; rr++) {
    const int r = cgp * 16 + rr;
    sacc += B[r + k * TB] * v[r];
  }
  part4[cgp][k] = sacc;
  __syncthreads();
  if (threadIdx.x < TB) {
    const int cc = threadIdx.x;
    if (cc < nr) y[r0 + cc] = part4[0][cc] + part4[1][cc] + part4[2][cc] + part4[3][cc];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicExch(&flags[i], 1);
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
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(k_inv_blocks, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * TB * (TB + 1) * 8);
      attr = true;
    }
    MDS_LAUNCH(PC_SOLVE_FWD, st,
               (k_inv_blocks<<<(unsigned)nblk, 256, 2 * TB * (TB + 1) * sizeof(double), st>>>(N, LD, ldm, s.binv)));
    MDS_LAUNCH(PC_SOLVE_FWD, st,
               (k_trsv_fwd<<<(unsigned)nblk, ST, 0, st>>>(N, LD, ldm, s.y, s.binv, s.flags, s.tickets)));
    const double* tolp = (zero_tol < 0.0 && fwork) ? mds_factor_tol_ptr(fwork) : nullptr;
    MDS_LAUNCH(PC_SOLVE_D, st,
               (k_dsolve<<<ge, 256, 0, st>>>(N, LD, ldm, piv, s.y, tolp, zero_tol < 0.0 ? 0.0 : zero_tol, status)));
    MDS_CUDA_TRY(cudaMemsetAsync(s.flags, 0, sizeof(int) * (nblk + 1), st));
    MDS_LAUNCH(PC_SOLVE_BWD, st,
               (k_trsv_bwd<<<(unsigned)nblk, ST, 0, st>>>(N, LD, ldm, s.y, s.binv, s.flags, s.tickets + 1)));
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
