// i8_umma_probe.cu -- standalone check of the tcgen05 INT8 MMA building blocks
// used by the emulated-FP64 trailing update: shared-memory (UMMA) descriptors
// for K-major int8 operands (no swizzle and 64-byte swizzle), the instruction
// descriptor of kind::i8 with S32 accumulation, TMEM alloc / ld, commit to an
// mbarrier.  One CTA computes D[128 x 64] = A[128 x 64] * B[64 x 64]^T (int8,
// K = 64 as two K = 32 instructions) and the host compares with a CPU product.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o i8_umma_probe i8_umma_probe.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// K-major canonical layouts (in bytes, 1-byte elements):
//   SWIZZLE_NONE: element (r, k) at (r/8)*SBO + (k/16)*LBO + (r%8)*16 + k%16
//   SWIZZLE_64B : rows of 64 bytes, 16-byte chunk index XORed with (r%8)/2 ... (Swizzle<2,4,3>:
//                 bits [4,6) ^= bits [7,9) of the byte offset), 8-row groups SBO apart
__host__ __device__ inline uint32_t off_none(int r, int k, int SBO, int LBO) {
  return (uint32_t)((r / 8) * SBO + (k / 16) * LBO + (r % 8) * 16 + (k % 16));
}
__host__ __device__ inline uint32_t off_sw64(int r, int k) {
  const uint32_t lin = (uint32_t)(r * 64 + k);
  return lin ^ (((lin >> 7) & 3u) << 4);
}

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;                       // version (sm_100)
  d |= (uint64_t)(layout & 7) << 61;
  return d;
}

template <int SW>
__global__ void __launch_bounds__(128) probe(const int8_t* A, const int8_t* B, int32_t* D) {
  __shared__ __align__(1024) int8_t sA[128 * 64];
  __shared__ __align__(1024) int8_t sB[64 * 64];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int SBO = SW ? 512 : 512, LBO = SW ? 16 : 128;
  for (int i = tid; i < 128 * 64; i += 128) {
    const int r = i / 64, k = i % 64;
    sA[SW ? off_sw64(r, k) : off_none(r, k, SBO, LBO)] = A[i];
  }
  for (int i = tid; i < 64 * 64; i += 128) {
    const int r = i / 64, k = i % 64;
    sB[SW ? off_sw64(r, k) : off_none(r, k, SBO, LBO)] = B[i];
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;\n" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");   // generic smem writes -> async proxy (MMA)
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = tmem_base;
  if (tid == 0) {
    // idesc: D = S32 (bits 4-5 = 2), A = B = S8 (bits 7-9, 10-12 = 1), K-major, N>>3 at 17, M>>4 at 24
    const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((64u >> 3) << 17) | ((128u >> 4) << 24);
    for (int kk = 0; kk < 2; kk++) {
      // K = 32 bytes per instruction: advance the start address by the K offset of the chunk pair
      const uint32_t koff = SW ? 32u * kk : 2u * LBO * kk;
      const uint64_t da = make_desc(smem_u32(sA) + koff, LBO, SBO, SW ? 4 : 0);
      const uint64_t db = make_desc(smem_u32(sB) + koff, LBO, SBO, SW ? 4 : 0);
      const uint32_t acc = kk > 0 ? 1u : 0u;
      asm volatile(
          "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
          " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
          "l"(da), "l"(db), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&bar))
                 : "memory");
  }
  // wait for the MMAs (phase 0)
  asm volatile(
      "{\n .reg .pred P1;\n WAIT:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n @!P1 bra WAIT;\n}\n" ::"r"(
          smem_u32(&bar)) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  // each warp reads its 32 TMEM lanes (rows), 64 columns
  uint32_t v[64];
  const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16);
#pragma unroll
  for (int c = 0; c < 64; c += 16) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
        : "=r"(v[c + 0]), "=r"(v[c + 1]), "=r"(v[c + 2]), "=r"(v[c + 3]), "=r"(v[c + 4]), "=r"(v[c + 5]),
          "=r"(v[c + 6]), "=r"(v[c + 7]), "=r"(v[c + 8]), "=r"(v[c + 9]), "=r"(v[c + 10]), "=r"(v[c + 11]),
          "=r"(v[c + 12]), "=r"(v[c + 13]), "=r"(v[c + 14]), "=r"(v[c + 15])
        : "r"(ta + c));
  }
  asm volatile("tcgen05.wait::ld.sync.aligned;\n");
  const int row = warp * 32 + lane;
  for (int c = 0; c < 64; c++) D[row * 64 + c] = (int32_t)v[c];
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;\n" ::"r"(tmem));
}

int main() {
  std::vector<int8_t> A(128 * 64), B(64 * 64);
  srand(1);
  for (auto& a : A) a = (int8_t)(rand() % 255 - 127);
  for (auto& b : B) b = (int8_t)(rand() % 255 - 127);
  std::vector<int32_t> ref(128 * 64);
  for (int i = 0; i < 128; i++)
    for (int j = 0; j < 64; j++) {
      int32_t s = 0;
      for (int k = 0; k < 64; k++) s += (int32_t)A[i * 64 + k] * (int32_t)B[j * 64 + k];
      ref[i * 64 + j] = s;
    }
  int8_t *dA, *dB;
  int32_t* dD;
  cudaMalloc(&dA, A.size());
  cudaMalloc(&dB, B.size());
  cudaMalloc(&dD, 128 * 64 * 4);
  cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
  int bad_total = 0;
  for (int sw = 0; sw < 2; sw++) {
    cudaMemset(dD, 0, 128 * 64 * 4);
    if (sw) probe<1><<<1, 128>>>(dA, dB, dD);
    else probe<0><<<1, 128>>>(dA, dB, dD);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<int32_t> D(128 * 64);
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int i = 0; i < 128 * 64; i++) bad += D[i] != ref[i];
    printf("swizzle %s: %s, mismatches %d / %d; D[0..3] = %d %d %d %d, ref = %d %d %d %d\n", sw ? "64B" : "none",
           cudaGetErrorString(e), bad, 128 * 64, D[0], D[1], D[2], D[3], ref[0], ref[1], ref[2], ref[3]);
    bad_total += bad + (e != cudaSuccess);
  }
  return bad_total ? 1 : 0;
}
