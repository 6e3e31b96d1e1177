// anorm.cuh — fixed-order ||M||_inf of a symmetric matrix stored as its lower
// triangle (row abs-sums via symmetry: row i = sum_{j<=i} |M(i,j)| +
// sum_{j>i} |M(j,i)|), plus a non-finite check (pre-factor scan, SURVEY §8(a3);
// tolerance tol = N eps ||M||_inf, reading R4; NaN/Inf -> NONFINITE, R17).
//
// The lower triangle is cut into 64x64 tiles (I, J), I >= J, id I(I+1)/2 + J.
// Whoever owns a tile's final values (the condensation epilogue, or the
// stand-alone scan below) writes two 64-vectors of partial sums:
//   prow[tile][r] = sum_{c: j <= i} |M(i, j)|   (i = 64I + r, j = 64J + c)
//   pcol[tile][c] = sum_{r: i >  j} |M(i, j)|
// each summed in a fixed order.  k_anorm_rows then forms, for every row i of
// block b,  rowsum(i) = sum_{J<=b} prow[(b,J)] + sum_{I>=b} pcol[(I,b)]  in a
// fixed order and max-reduces (max is exact).  So ||M||_inf is deterministic
// (bitwise reproducible run to run and across batch positions), unlike an
// atomic-add row sum.  Product path only (not shared with oracle/).
#pragma once
#include "common.cuh"

namespace {   // internal linkage: included by several translation units
namespace anorm {

constexpr int AT = 64;    // tile edge
constexpr int AW = 8;     // warps per CTA of the tile owners

__host__ __device__ inline int64_t ntiles(int64_t N) {
  const int64_t nb = (N + AT - 1) / AT;
  return nb * (nb + 1) / 2;
}
__host__ __device__ inline int64_t tile_id(int64_t I, int64_t J) { return I * (I + 1) / 2 + J; }

// ctr[0] tile queue, ctr[1] ticket of k_anorm_rows, ctr[2] non-finite flag, ctr[3] spare
struct Parts {
  double* prow;      // [ntiles * 64]
  double* pcol;      // [ntiles * 64]
  double* bmax;      // [ceil(N/256)]
  unsigned* ctr;     // [4]
};

inline size_t parts_bytes(int64_t N) {
  const int64_t nt = ntiles(N);
  return (((size_t)nt * AT * 16 + (size_t)((N + 31) / 32 + 1) * 8 + 64) + 255) / 256 * 256;
}

// the Parts of one matrix inside a block of parts_bytes(N) bytes at `base`
__host__ __device__ inline Parts parts_at(char* base, int64_t N) {
  const int64_t nt = ntiles(N);
  Parts P;
  P.prow = reinterpret_cast<double*>(base);
  P.pcol = P.prow + nt * AT;
  P.bmax = P.pcol + nt * AT;
  P.ctr = reinterpret_cast<unsigned*>(P.bmax + (N + 31) / 32 + 1);
  return P;
}

// Outputs of k_anorm_rows for matrix s = blockIdx.y (batched: one launch for
// all matrices).  anorm[s] (elements); tol / abort at byte offset s * ctl_stride
// from tol0 / abort0 (NULL: not written); status + s * status_stride.
struct NormOut {
  double* anorm;
  double* tol0;
  int* abort0;
  size_t ctl_stride;
  int32_t* status;
  int64_t status_stride;
  double zero_tol;
  const int32_t* active;   // [batch] or NULL: matrices with active[s] == 0 are skipped
};

// Per-thread share of a tile's partials.  Thread layout used by every owner:
// warp w holds columns c = w + 8u (u = 0..7), lane l holds rows l and l + 32.
// v[u][h] is the value at (row l + 32h, column w + 8u) (0 when outside the
// lower triangle or the matrix).  red: __shared__ double[AW][64].
__device__ __forceinline__ void tile_partials(const double (&v)[8][2], const bool (&strict)[8][2], int64_t tile,
                                              const Parts& P, double (*red)[AT]) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double ra[2] = {0.0, 0.0};
#pragma unroll
  for (int u = 0; u < 8; u++) {
    const double a0 = fabs(v[u][0]), a1 = fabs(v[u][1]);
    ra[0] += a0;
    ra[1] += a1;
    double cs = (strict[u][0] ? a0 : 0.0) + (strict[u][1] ? a1 : 0.0);
    cs = warp_sum(cs);
    if (lane == 0) P.pcol[tile * AT + warp + 8 * u] = cs;
  }
  red[warp][lane] = ra[0];
  red[warp][lane + 32] = ra[1];
  __syncthreads();
  if (threadIdx.x < AT) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < AW; w++) s += red[w][threadIdx.x];
    P.prow[tile * AT + threadIdx.x] = s;
  }
}

// Row sums from the partials (fixed order), block max, and -- in the last CTA
// of matrix s = blockIdx.y to finish (ticket) -- the global max into
// anorm[s] (NaN if a non-finite entry was seen).  When tol0 != NULL also sets
// the tolerance (zero_tol < 0: N eps ||M||_inf, else zero_tol) and, on a
// non-finite matrix, abort = 1 and status NONFINITE.  Resets the ticket.
// A CTA takes 32 rows (lane = row); row i of block b has nb + 1 partials
// (prow of tiles (b, 0..b), then pcol of tiles (b..nb-1, b)), split into 8
// fixed ranges, one per warp, summed in order and then combined in warp order.
__global__ void __launch_bounds__(256) k_anorm_rows(int64_t N, char* parts, size_t parts_stride, NormOut o) {
  pdl_wait();
  pdl_trigger();
  const int64_t ms = blockIdx.y;
  if (o.active && !o.active[ms]) return;
  const Parts P = parts_at(parts + ms * parts_stride, N);
  const int64_t nb = (N + AT - 1) / AT;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t i = blockIdx.x * 32ll + lane;
  __shared__ double part[AW][32];
  double s = 0.0;
  if (i < N) {
    const int64_t b = i / AT, r = i % AT;
    const int64_t nterm = nb + 1, per = (nterm + AW - 1) / AW;
    const int64_t x0 = min(nterm, per * warp), x1 = min(nterm, per * (warp + 1));
    constexpr int CH = 8;   // loads issued ahead of the (in-order) sum
    for (int64_t x = x0; x < x1; x += CH) {
      double t[CH];
#pragma unroll
      for (int q = 0; q < CH; q++) {
        const int64_t xq = x + q;
        t[q] = xq < x1 ? ((xq <= b) ? P.prow[tile_id(b, xq) * AT + r] : P.pcol[tile_id(xq - 1, b) * AT + r]) : 0.0;
      }
#pragma unroll
      for (int q = 0; q < CH; q++)
        if (x + q < x1) s += t[q];
    }
  }
  part[warp][lane] = s;
  __syncthreads();
  __shared__ bool last;
  if (warp == 0) {
    double rs = 0.0;
#pragma unroll
    for (int w = 0; w < AW; w++) rs += part[w][lane];
    rs = warp_max(rs);
    if (lane == 0) {
      P.bmax[blockIdx.x] = rs;
      __threadfence();
      last = atomicAdd(&P.ctr[1], 1u) == gridDim.x - 1;
    }
  }
  __syncthreads();
  if (last && warp == 0) {
    __threadfence();
    double a = 0.0;   // max is exact: any order
    for (unsigned b = lane; b < gridDim.x; b += 32) a = fmax(a, *(volatile double*)&P.bmax[b]);
    a = warp_max(a);
    if (lane == 0) {
    const bool bad = *(volatile unsigned*)&P.ctr[2] != 0u || !isfinite(a);
    if (bad) a = __longlong_as_double(0x7ff8000000000000ll);   // NaN: "not finite"
    if (o.anorm) o.anorm[ms] = a;
    if (o.tol0) {
      double* tol = reinterpret_cast<double*>(reinterpret_cast<char*>(o.tol0) + ms * o.ctl_stride);
      *tol = o.zero_tol < 0.0 ? (double)N * 2.220446049250313e-16 * a : o.zero_tol;
      if (bad) {
        if (o.abort0) *reinterpret_cast<int*>(reinterpret_cast<char*>(o.abort0) + ms * o.ctl_stride) = 1;
        if (o.status) mds_set_status(o.status + ms * o.status_stride, MDS_ERR_NONFINITE);
      }
    }
    P.ctr[1] = 0u;
    P.ctr[2] = 0u;
    }
  }
}

// launch k_anorm_rows for `batch` matrices (partials `parts_stride` bytes apart)
inline cudaError_t launch_rows(int64_t N, char* parts, size_t parts_stride, const NormOut& o, int64_t batch,
                               cudaStream_t st) {
  return launch_pdl(k_anorm_rows, dim3((unsigned)((N + 31) / 32), (unsigned)batch), dim3(256), 0, st, N, parts,
                    parts_stride, o);
}

// Stand-alone scan of a matrix already in memory (mds_factor without a
// condensation-provided norm): one CTA per lower tile, read once.
// Batched: matrix s = blockIdx.y at A + s * a_stride, partials at parts + s * parts_stride.
__global__ void __launch_bounds__(256) k_anorm_scan(int64_t N, const double* __restrict__ A, int64_t lda,
                                                    int64_t a_stride, char* parts, size_t parts_stride) {
  pdl_wait();
  pdl_trigger();
  A += blockIdx.y * a_stride;
  const Parts P = parts_at(parts + blockIdx.y * parts_stride, N);
  __shared__ double red[AW][AT];
  const int64_t t = blockIdx.x;
  int64_t I = (int64_t)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
  while (I * (I + 1) / 2 > t) I--;
  while ((I + 1) * (I + 2) / 2 <= t) I++;
  const int64_t J = t - I * (I + 1) / 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double v[8][2];
  bool strict[8][2];
  bool bad = false;
#pragma unroll
  for (int u = 0; u < 8; u++) {
    const int64_t j = J * AT + warp + 8 * u;
#pragma unroll
    for (int h = 0; h < 2; h++) {
      const int64_t i = I * AT + lane + 32 * h;
      const bool in = i < N && j < N && i >= j;
      v[u][h] = in ? A[i + j * lda] : 0.0;
      strict[u][h] = in && i > j;
      if (!isfinite(v[u][h])) bad = true;
    }
  }
  if (bad) atomicOr(&P.ctr[2], 1u);
  tile_partials(v, strict, t, P, red);
}

}  // namespace anorm
}  // namespace
