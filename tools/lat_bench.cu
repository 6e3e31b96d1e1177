// dependent-chain latency microbenchmarks (cycles per op) for the panel critical path
#include <cstdio>
__global__ void k(double* out, long long* t, double a0) {
  double x = a0 + threadIdx.x * 1e-9;
  long long c0, c1;
  // DFMA chain
  c0 = clock64();
  #pragma unroll 1
  for (int i = 0; i < 1000; i++) x = fma(x, 0.999999, 1e-7);
  c1 = clock64(); if (threadIdx.x == 0) t[0] = (c1 - c0);
  // rcp.approx chain
  c0 = clock64();
  #pragma unroll 1
  for (int i = 0; i < 1000; i++) { double r; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); x = r; }
  c1 = clock64(); if (threadIdx.x == 0) t[1] = (c1 - c0);
  // shfl chain (double)
  c0 = clock64();
  #pragma unroll 1
  for (int i = 0; i < 1000; i++) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31);
  c1 = clock64(); if (threadIdx.x == 0) t[2] = (c1 - c0);
  // full-precision division chain
  c0 = clock64();
  #pragma unroll 1
  for (int i = 0; i < 1000; i++) x = 1.0 / (x + 1.0);
  c1 = clock64(); if (threadIdx.x == 0) t[3] = (c1 - c0);
  // DMUL chain
  c0 = clock64();
  #pragma unroll 1
  for (int i = 0; i < 1000; i++) x = x * 1.0000001;
  c1 = clock64(); if (threadIdx.x == 0) t[4] = (c1 - c0);
  out[threadIdx.x] = x;
}
__global__ void ks(double* out, long long* t) {
  __shared__ double sm[256];
  sm[threadIdx.x] = threadIdx.x;
  __syncthreads();
  long long c0 = clock64();
  double x = 0;
  #pragma unroll 1
  for (int i = 0; i < 1000; i++) { __syncthreads(); x += sm[(threadIdx.x + i) & 63]; }
  long long c1 = clock64(); if (threadIdx.x == 0) t[5] = c1 - c0;
  out[threadIdx.x] = x;
}
int main() {
  double* o; long long* t; cudaMalloc(&o, 8192); cudaMalloc(&t, 64);
  k<<<1, 32>>>(o, t, 1.5); ks<<<1, 256>>>(o, t); cudaDeviceSynchronize();
  k<<<1, 32>>>(o, t, 1.5); ks<<<1, 256>>>(o, t); cudaDeviceSynchronize();
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  long long h[8]; cudaMemcpy(h, t, 48, cudaMemcpyDeviceToHost);
  printf("cycles/op: DFMA %.1f  RCP64 %.1f  SHFL %.1f  DIV %.1f  DMUL %.1f  syncthreads+LDS(256thr) %.1f\n",
         h[0] / 1000.0, h[1] / 1000.0, h[2] / 1000.0, h[3] / 1000.0, h[4] / 1000.0, h[5] / 1000.0);
}
