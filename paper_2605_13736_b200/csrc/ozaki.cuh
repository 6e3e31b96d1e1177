// ozaki.cuh — the trailing update C -= L21 W21^T of the BK factorization in
// emulated FP64 on the INT8 tensor cores (Ozaki-scheme
// error-free splitting), included by factor.cu.
//
// Splitting (k_oz_split, once per panel): every row r of the panel's L (Lb) and
// W buffers (kb <= 64 columns, zero beyond) is scaled by 2^-e_r, e_r the frexp
// exponent of the row's max |entry|, so x = v 2^-e_r lies in (-1, 1), and cut
// into 8 signed 7-bit slices by exact steps y = 128 x, q = trunc(y), x = y - q:
//   v = 2^e_r (sum_{i<8} q_i 2^{-7(i+1)} + 2^{-56} x_8),  |q_i| <= 127.
// The product (L W^T)[r, c] = 2^{e_r + f_c} sum_{i,j} 2^{-7(i+j+2)} (Q^L_i Q^W_j^T)[r, c],
// and every Q^L_i Q^W_j^T (K = 64, |.| < 2^20) is EXACT in int32 on the tensor
// cores (tcgen05.mma kind::i8, S32 accumulators in TMEM).  Terms with
// s = i + j <= 7 are kept (36 products, summed per level s in TMEM: |D_s| < 2^24);
// the dropped ones and the slicing tail are below 2^-46.8 and 2^-49 of
// 2^{e_r + f_c}, inside the FP64 GEMM error bound gamma_64 sum |l||w| <= 2^-41
// of it.  The epilogue combines the 8 levels EXACTLY in two int64 sums
//   hi = sum_{s<4} D_s 2^{7(3-s)},  lo = sum_{s>=4} D_s 2^{7(7-s)}   (|.| < 2^45)
// and forms T = 2^{E-35} hi + 2^{E-63} lo (E = e_r + f_c; two exact int64 ->
// double conversions, one rounding), then -T is TMA-reduce-added into M.
//
// Kernel shape: one CTA = 1 producer/MMA warp + 4 epilogue warps (TMEM lane
// quadrants), 128 x 32 output tiles, the 8 L slices (8 x 8 KB) and 8 W slices
// (8 x 2 KB) of a tile in one 64-byte-swizzled stage (TMA), 256 TMEM columns
// (8 levels x 32), two CTAs per SM so one CTA's MMAs overlap the other's
// epilogue.  Tile queue: 128-row blocks I >= J of the trailing lower triangle,
// 4 column quarters each; batched: slot = scenario * tiles + tile (3-D maps).
#pragma once

namespace {
constexpr int OZ_S = 8;                        // slices per operand
constexpr int OZ_TM = 128, OZ_TN = 32;         // output tile
constexpr int OZ_LB = OZ_TM * 64;              // bytes per L slice tile (8 KB)
constexpr int OZ_WB = OZ_TN * 64;              // bytes per W slice tile (2 KB)
constexpr int OZ_STAGE = OZ_S * (OZ_LB + OZ_WB);
constexpr int OZ_TMEM_COLS = OZ_S * OZ_TN;     // 256

// ---------------------------------------------------------------------------
// split: rows [r_lo, N) of the panel's L (Lb) and W into slices
// ozL/ozW[(8 s + i) * N * 64 + r * 64 + k] (int8) and exponents ozeL/ozeW[r].
// Rows below the panel (r < k0) are zero.  One CTA = 64 rows x 64 columns.
__global__ void __launch_bounds__(256) k_oz_split(int64_t N, FWork f, int64_t r_lo) {
  pdl_wait();
  pdl_trigger();
  bsel_ws(f, blockIdx.z);
  if (f.ctl->abort) return;
  const int2 pi = f.pinfo[f.pidx];
  const int64_t k0 = pi.x;
  const int kb = pi.y;
  const int64_t r0 = r_lo + blockIdx.x * 64ll;
  if (r0 >= N) return;
  const bool isW = blockIdx.y == 1;
  const double* src = isW ? f.W : f.Lb;
  int8_t* dst = isW ? f.ozW : f.ozL;
  int* dexp = isW ? f.ozeW : f.ozeL;
  __shared__ double t[64][65];
  const int tid = threadIdx.x;
  for (int idx = tid; idx < 64 * 64; idx += 256) {
    const int r = idx & 63, k = idx >> 6;
    const int64_t row = r0 + r;
    t[r][k] = (row < N && row >= k0 && k < kb) ? src[row + (int64_t)k * f.ldw] : 0.0;
  }
  __syncthreads();
  const int warp = tid >> 5, lane = tid & 31;
  for (int r = warp; r < 64; r += 8) {
    const int64_t row = r0 + r;
    if (row >= N) break;
    double a = t[r][2 * lane], b = t[r][2 * lane + 1];
    double mx = fmax(fabs(a), fabs(b));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    int e = 0;
    if (mx > 0.0 && isfinite(mx)) (void)frexp(mx, &e);
    if (lane == 0) dexp[row] = e;
    a = scalbn(a, -e);
    b = scalbn(b, -e);
#pragma unroll
    for (int i = 0; i < OZ_S; i++) {
      const double ya = a * 128.0, yb = b * 128.0;   // exact (power-of-two scaling)
      const double qa = trunc(ya), qb = trunc(yb);
      a = ya - qa;                                   // exact
      b = yb - qb;
      const int ia = (int)qa, ib = (int)qb;
      const unsigned short pk = (unsigned short)((ia & 0xff) | ((ib & 0xff) << 8));
      *reinterpret_cast<unsigned short*>(dst + ((int64_t)i * N + row) * 64 + 2 * lane) = pk;
    }
  }
}

__device__ __forceinline__ void tma_load_4d(unsigned dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                            unsigned bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];\n" ::"r"(dst),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar)
      : "memory");
}
__device__ __forceinline__ uint64_t oz_desc(uint32_t saddr) {   // K-major, 64-byte swizzle, 8-row groups 512 B apart
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;             // LBO (unused for swizzled K-major)
  d |= (uint64_t)(512 >> 4) << 32;    // SBO
  d |= (uint64_t)1 << 46;             // version
  d |= (uint64_t)4 << 61;             // SWIZZLE_64B
  return d;
}
__device__ __forceinline__ double oz_pow2(int k) {   // 2^k for |k| <= 2044 (product of two normal powers)
  const int h = k / 2, l = k - h;
  auto p = [](int x) {
    x = x < -1022 ? -1022 : (x > 1023 ? 1023 : x);
    return __longlong_as_double((long long)(x + 1023) << 52);
  };
  return p(h) * p(l);
}

// Tile decode: local index x -> (128-row block I, 128-column block J <= I, quarter t) of
// the trailing lower triangle starting at block ib0; returns false if the quarter holds no
// column >= s or lies beyond N.
__device__ __forceinline__ bool oz_tile(int64_t x, int64_t N, int64_t s, int64_t& R0, int64_t& C0) {
  const int64_t ib0 = s / OZ_TM;
  int64_t bi, bj;
  tri_tile(x >> 2, bi, bj);
  R0 = (ib0 + bi) * OZ_TM;
  C0 = (ib0 + bj) * OZ_TM + (x & 3) * OZ_TN;
  return C0 < N && C0 + OZ_TN > s && R0 < N;
}

// BT: batched (slot = scenario * bt_tiles + item).  Maps: mapOL / mapOW int8 slices, dims
// {64, N, 8, batch}, boxes {64, 128 | 32, 1, 1}, 64-byte swizzle; mapC FP64 M, dims {N, N, batch},
// box {128, 32, 1}, no swizzle (the reduce-add target).
// Work item = one 128 x 128 block (I, J) of the trailing lower triangle: its 8 L slice tiles
// (64 KB) are loaded ONCE and stay in shared memory while the block's four 32-column quarters
// stream through (8 W slice tiles, 16 KB each) -- 8 B of operands per output instead of 20.
// Warp roles (one CTA per SM): warp 0 producer (TMA; 2 L stages, 2 W stages), warp 1 MMA
// issuer (72 tcgen05.mma per quarter into one of 2 TMEM buffers of 8 x 32 columns), warps 2-5
// epilogue (TMEM lane quadrant warp % 4): exact int64 level combination, scaling, -T into a
// staging tile, TMA reduce-add.  Every hand-off is an mbarrier (tcgen05.commit for the MMA
// side), so loads, MMAs and epilogues of consecutive quarters overlap.
constexpr int OZ_THREADS2 = 192;
constexpr int OZ_STG = OZ_TM * OZ_TN * 8;                    // FP64 staging tile (32 KB)
constexpr int OZ_LST = OZ_S * OZ_LB;                         // L stage (64 KB)
constexpr int OZ_WST = OZ_S * OZ_WB;                         // W stage (16 KB)
constexpr int OZ_NWS = 4;                                    // W stages
constexpr int OZ_SMEM2 = 2 * OZ_LST + OZ_NWS * OZ_WST + OZ_STG + 1024 + 768;
template <bool BT>
__global__ void __launch_bounds__(OZ_THREADS2, 1) k_update_oz(int64_t N, FWork f,
                                                           const __grid_constant__ CUtensorMap mapOL,
                                                           const __grid_constant__ CUtensorMap mapOW,
                                                           const __grid_constant__ CUtensorMap mapC,
                                                           int64_t bt_tiles, int64_t bt_n) {
  extern __shared__ unsigned char ozsm_raw[];
  const unsigned base = (smem_u32(ozsm_raw) + 1023u) & ~1023u;
  unsigned char* gbase = ozsm_raw + (base - smem_u32(ozsm_raw));
  const unsigned sLb = base, sWb = base + 2 * OZ_LST;
  const unsigned stg_s = sWb + OZ_NWS * OZ_WST;                // staging tile (shared-window address)
  double* stg = reinterpret_cast<double*>(gbase + (stg_s - base));
  const unsigned bars = stg_s + OZ_STG;
  // lfull[2], lempty[2], wfull[4], wempty[4], tfull[2], tempty[2] (4 slots per kind)
  auto bar = [&](int kind, int i) { return bars + 32 * kind + 8 * i; };
  volatile long long* islot = reinterpret_cast<volatile long long*>(gbase + (bars - base) + 192);   // [2][2] per L stage
  volatile long long* tslot = islot + 4;                                                           // [2][2] per TMEM buffer
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(gbase + (bars - base) + 256);
  double* cscale = reinterpret_cast<double*>(gbase + (bars - base) + 264);                          // [32]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int k = 0; k < 6; k++)
      for (int i = 0; i < 4; i++) mbar_init(bar(k, i), 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                 "n"(2 * OZ_TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = *tmem_slot;
  unsigned long long* counter = f.ucount + 3 * f.pidx;
  constexpr int LFULL = 0, LEMPTY = 1, WFULL = 2, WEMPTY = 3, TFULL = 4, TEMPTY = 5;
  if (warp == 0) {
    // ---------------- producer
    if (lane == 0) {
      int64_t s_single = 0;
      if (!BT) {
        const int2 pi = f.pinfo[f.pidx];
        s_single = (int64_t)pi.x + pi.y;
      }
      const int64_t nall = BT ? bt_n * bt_tiles : bt_tiles;
      int wq = 0;                                   // quarters produced so far (W stage / phase)
      for (int it = 0;; it++) {
        const int ls = it & 1;
        if (it >= 2) mbar_wait(bar(LEMPTY, ls), ((it >> 1) - 1) & 1);
        int64_t R0 = -1, C0 = 0, sc = 0, sT = s_single;
        for (;;) {
          const unsigned long long x = atom_add_u64(counter, 1ull);
          if (x >= (unsigned long long)nall) break;
          int64_t lt = (int64_t)x;
          if (BT) {
            sc = (int64_t)(x / (unsigned long long)bt_tiles);
            lt = (int64_t)(x % (unsigned long long)bt_tiles);
            const size_t bo = (size_t)sc * f.bws;
            const FCtl* cs = reinterpret_cast<const FCtl*>(reinterpret_cast<const char*>(f.ctl) + bo);
            if (cs->abort) continue;
            const int2 ps = reinterpret_cast<const int2*>(reinterpret_cast<const char*>(f.pinfo) + bo)[f.pidx];
            if (ps.y <= 0) continue;
            sT = (int64_t)ps.x + ps.y;
          } else if (f.ctl->abort) {
            break;
          }
          if (N - sT <= 0) continue;
          const int64_t ib0 = sT / OZ_TM;
          int64_t bi, bj;
          tri_tile(lt, bi, bj);
          if ((ib0 + bi) * OZ_TM >= N) continue;
          R0 = (ib0 + bi) * OZ_TM;
          C0 = (ib0 + bj) * OZ_TM;
          break;
        }
        if (R0 < 0) {
          islot[2 * ls] = -1;
          mbar_arrive(bar(LFULL, ls));
          break;
        }
        islot[2 * ls] = (long long)(((unsigned long long)C0 << 32) | (unsigned long long)R0);
        islot[2 * ls + 1] = (long long)(((unsigned long long)sc << 32) | (unsigned long long)sT);
        const unsigned sL = sLb + ls * OZ_LST;
        mbar_expect_tx(bar(LFULL, ls), OZ_LST);
#pragma unroll
        for (int i = 0; i < OZ_S; i++) tma_load_4d(sL + i * OZ_LB, &mapOL, 0, (int)R0, i, (int)sc, bar(LFULL, ls));
        for (int q = 0; q < 4; q++, wq++) {
          const int ws = wq % OZ_NWS;
          if (wq >= OZ_NWS) mbar_wait(bar(WEMPTY, ws), ((wq / OZ_NWS) - 1) & 1);
          const unsigned sW = sWb + ws * OZ_WST;
          mbar_expect_tx(bar(WFULL, ws), OZ_WST);
#pragma unroll
          for (int i = 0; i < OZ_S; i++)
            tma_load_4d(sW + i * OZ_WB, &mapOW, 0, (int)(C0 + q * OZ_TN), i, (int)sc, bar(WFULL, ws));
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer
    if (lane == 0) {
      const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(OZ_TN >> 3) << 17) |
                             ((uint32_t)(OZ_TM >> 4) << 24);
      int wq = 0;
      for (int it = 0;; it++) {
        const int ls = it & 1;
        mbar_wait(bar(LFULL, ls), (it >> 1) & 1);
        const long long x0 = islot[2 * ls], x1 = islot[2 * ls + 1];
        if (x0 == -1) {
          const int tb = wq & 1;
          if (wq >= 2) mbar_wait(bar(TEMPTY, tb), ((wq >> 1) - 1) & 1);
          tslot[2 * tb] = -1;
          mbar_arrive(bar(TFULL, tb));
          break;
        }
        const unsigned sL = sLb + ls * OZ_LST;
        for (int q = 0; q < 4; q++, wq++) {
          const int ws = wq % OZ_NWS, tb = wq & 1;
          mbar_wait(bar(WFULL, ws), (wq / OZ_NWS) & 1);
          if (wq >= 2) mbar_wait(bar(TEMPTY, tb), ((wq >> 1) - 1) & 1);   // epilogue done with this buffer
          tslot[2 * tb] = (long long)((unsigned long long)x0 + ((unsigned long long)(q * OZ_TN) << 32));
          tslot[2 * tb + 1] = x1;
          asm volatile("tcgen05.fence::after_thread_sync;\n");
          const unsigned sW = sWb + ws * OZ_WST;
          const uint32_t tacc = tmem + (uint32_t)(tb * OZ_TMEM_COLS);
          bool first[OZ_S];
#pragma unroll
          for (int v = 0; v < OZ_S; v++) first[v] = true;
#pragma unroll
          for (int i = 0; i < OZ_S; i++) {
#pragma unroll
            for (int j = 0; j < OZ_S; j++) {
              if (i + j >= OZ_S) continue;
              const int lv = i + j;
#pragma unroll
              for (int kk = 0; kk < 2; kk++) {
                const uint64_t da = oz_desc(sL + i * OZ_LB + 32 * kk);
                const uint64_t db = oz_desc(sW + j * OZ_WB + 32 * kk);
                const uint32_t acc = first[lv] ? 0u : 1u;
                first[lv] = false;
                asm volatile(
                    "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                    " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tacc + (uint32_t)(lv * OZ_TN)),
                    "l"(da), "l"(db), "r"(idesc), "r"(acc));
              }
            }
          }
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                           bar(WEMPTY, ws))
                       : "memory");
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                           bar(TFULL, tb))
                       : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                         bar(LEMPTY, ls))
                     : "memory");
      }
    }
  } else {
    // ---------------- epilogue: warp w reads TMEM lanes 32 (w % 4) .. +31 = output rows of the tile
    const int qd = warp & 3;
    const int rl = qd * 32 + lane;
    const int et = threadIdx.x - 64;               // 0..127
    for (int it = 0;; it++) {
      const int tb = it & 1;
      mbar_wait(bar(TFULL, tb), (it >> 1) & 1);
      const long long x0 = tslot[2 * tb];
      if (x0 == -1) break;
      asm volatile("tcgen05.fence::after_thread_sync;\n");
      const int64_t R0 = (int64_t)(unsigned)(x0 & 0xffffffffll), C0 = (int64_t)(x0 >> 32);
      const long long x1 = tslot[2 * tb + 1];
      const int64_t sc = (int64_t)(x1 >> 32), sT = (int64_t)(x1 & 0xffffffffll);
      const bool live = C0 < N && C0 + OZ_TN > sT;   // a quarter left of the trailing matrix adds nothing
      const size_t bo = BT ? (size_t)sc * f.bws : 0;
      const int* eL = reinterpret_cast<const int*>(reinterpret_cast<const char*>(f.ozeL) + bo);
      const int* eW = reinterpret_cast<const int*>(reinterpret_cast<const char*>(f.ozeW) + bo);
      if (live) {
        // the previous quarter's reduce has read the staging tile; column scales of this quarter
        if (et == 0) asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
        if (et < OZ_TN) cscale[et] = (C0 + et < N) ? oz_pow2(eW[C0 + et]) : 0.0;
        asm volatile("bar.sync 1, 128;\n" ::: "memory");
        const int64_t row = R0 + rl;
        const double rscale = (row < N) ? oz_pow2(eL[row] - 35) : 0.0;
        const uint32_t ta = tmem + (uint32_t)(tb * OZ_TMEM_COLS) + ((uint32_t)(qd * 32) << 16);
#pragma unroll 1
        for (int c0 = 0; c0 < OZ_TN; c0 += 8) {
          uint32_t v[OZ_S][8];
#pragma unroll
          for (int lv = 0; lv < OZ_S; lv++)
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                         : "=r"(v[lv][0]), "=r"(v[lv][1]), "=r"(v[lv][2]), "=r"(v[lv][3]), "=r"(v[lv][4]),
                           "=r"(v[lv][5]), "=r"(v[lv][6]), "=r"(v[lv][7])
                         : "r"(ta + (uint32_t)(lv * OZ_TN + c0)));
          asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
          for (int c = 0; c < 8; c++) {
            long long hi = 0, lo = 0;
#pragma unroll
            for (int lv = 0; lv < 4; lv++) hi = hi * 128 + (long long)(int)v[lv][c];
#pragma unroll
            for (int lv = 4; lv < OZ_S; lv++) lo = lo * 128 + (long long)(int)v[lv][c];
            const int64_t col = C0 + c0 + c;
            // T = 2^{e_r + f_c} (2^-35 hi + 2^-63 lo) = (hi + 2^-28 lo) 2^{e_r - 35} 2^{f_c}
            const double u = fma((double)lo, 3.7252902984619140625e-09, (double)hi);
            const double T = u * rscale * cscale[c0 + c];
            const bool upd = row < N && row >= col && col >= sT;
            stg[(c0 + c) * OZ_TM + rl] = upd ? dneg(T) : 0.0;
          }
        }
      }
      // all TMEM reads of this buffer done -> MMA issuer; staging written -> TMA reduce-add
      asm volatile("tcgen05.fence::before_thread_sync;\n");
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      asm volatile("bar.sync 1, 128;\n" ::: "memory");
      if (et == 0) {
        mbar_arrive(bar(TEMPTY, tb));
        if (live) {
          asm volatile(
              "cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.tile.bulk_group [%0, {%1, %2, %3}], [%4];\n" ::"l"(
                  &mapC),
              "r"((int)R0), "r"((int)C0), "r"((int)sc), "r"(stg_s)
              : "memory");
          asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
        }
      }
    }
    if (et == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(2 * OZ_TMEM_COLS));
}

// int8 slice map: dims {64, N, 8, batch} (scenario blocks bws bytes apart), box {64, rows, 1, 1},
// 64-byte swizzle
bool make_map_oz(CUtensorMap* m, const int8_t* base, int64_t N, int64_t batch, size_t bws, int rows) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[4] = {64, (cuuint64_t)N, (cuuint64_t)OZ_S, (cuuint64_t)batch};
  cuuint64_t strides[3] = {64, (cuuint64_t)N * 64, (cuuint64_t)(bws ? bws : (size_t)N * 64 * OZ_S)};
  cuuint32_t box[4] = {64, (cuuint32_t)rows, 1, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<int8_t*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
// FP64 reduce-add target: dims {N, N, batch}, box {128, 32, 1}, no swizzle
bool make_map_ozc(CUtensorMap* m, const double* M, int64_t N, int64_t ldm, int64_t batch, size_t bstride) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[3] = {(cuuint64_t)N, (cuuint64_t)N, (cuuint64_t)batch};
  cuuint64_t strides[2] = {(cuuint64_t)ldm * 8, (cuuint64_t)bstride};
  cuuint32_t box[3] = {OZ_TM, OZ_TN, 1};
  cuuint32_t es[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(M), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
// work items (128 x 128 blocks) of one scenario whose trailing start is at least smin (queue bound)
int64_t oz_tiles(int64_t N, int64_t smin) {
  const int64_t nb = (N + OZ_TM - 1) / OZ_TM - smin / OZ_TM;
  return nb > 0 ? nb * (nb + 1) / 2 : 0;
}
}  // namespace
