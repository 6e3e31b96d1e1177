// FP64 ceiling microbenchmarks for the roofline denominator.
// DMMA: register-resident mma.sync.m8n8k4.f64 chains; DFMA: register-resident fma chains.
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS>
__global__ void dmma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[CHAINS][2];
#pragma unroll
  for (int i = 0; i < CHAINS; i++) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < CHAINS; i++) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; i++) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[0] = s;
}

template <int CHAINS>
__global__ void dmma16_loop(double* out, int iters) {
  // m16n8k16 f64: A 8 regs, B 4 regs, C 4 regs per thread
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; i++) a[i] = 1.0 + (threadIdx.x + i) * 1e-9;
#pragma unroll
  for (int i = 0; i < 4; i++) b[i] = 1.0 - (threadIdx.x + i) * 1e-9;
  double c[CHAINS][4];
#pragma unroll
  for (int i = 0; i < CHAINS; i++) for (int j = 0; j < 4; j++) c[i][j] = 0;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < CHAINS; i++) {
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; i++) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.0) out[0] = s;
}

template <int CHAINS>
__global__ void dfma_loop(double* out, int iters) {
  double x[CHAINS];
  double a = 1.0 + threadIdx.x * 1e-12, b = 1e-7;
#pragma unroll
  for (int i = 0; i < CHAINS; i++) x[i] = i;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < CHAINS; i++) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; i++) s += x[i];
  if (s == 12345.0) out[0] = s;
}

template <typename K>
double run(K kern, int blocks, int threads, int iters, double flops_per_thread_iter, const char* name) {
  double* d; cudaMalloc(&d, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  kern<<<blocks, threads>>>(d, iters / 10);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; r++) {
    cudaEventRecord(e0);
    kern<<<blocks, threads>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  double tf = (double)blocks * threads * iters * flops_per_thread_iter / (best * 1e-3) / 1e12;
  printf("{\"kernel\": \"%s\", \"blocks\": %d, \"threads\": %d, \"ms\": %.4f, \"tflops\": %.3f}\n", name, blocks, threads, best, tf);
  cudaFree(d);
  return tf;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int it = 2000;
  // m8n8k4: 2*8*8*4 = 512 flop per warp instr -> 16 per thread per mma
  run(dmma_loop<4>, sms * 4, 256, it, 4 * 16.0, "dmma_m8n8k4_c4_occ4x256");
  run(dmma_loop<8>, sms * 4, 256, it, 8 * 16.0, "dmma_m8n8k4_c8_occ4x256");
  run(dmma_loop<8>, sms * 2, 512, it, 8 * 16.0, "dmma_m8n8k4_c8_occ2x512");
  run(dmma_loop<8>, sms, 128, it, 8 * 16.0, "dmma_m8n8k4_c8_1x128");
  run(dmma_loop<8>, sms, 256, it, 8 * 16.0, "dmma_m8n8k4_c8_1x256");
  // m16n8k16: 2*16*8*16 = 4096 per warp instr -> 128 per thread
  run(dmma16_loop<2>, sms * 4, 256, it / 4, 2 * 128.0, "dmma_m16n8k16_c2_occ4x256");
  run(dmma16_loop<4>, sms * 2, 256, it / 4, 4 * 128.0, "dmma_m16n8k16_c4_occ2x256");
  run(dfma_loop<8>, sms * 4, 256, it, 8 * 2.0, "dfma_c8_occ4x256");
  run(dfma_loop<16>, sms * 4, 256, it, 16 * 2.0, "dfma_c16_occ4x256");
  return 0;
}
