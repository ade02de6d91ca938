// Micro-benchmark: dependent-chain latency (cycles/op) of FP64 ops and shuffles
// on one warp.  Diagnostics only.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, double seed, int n) {
  double x = seed + threadIdx.x * 1e-9, y = 1.0000001;
  long long t0, t1;
  const int N = 256;
  // DFMA chain
  t0 = clock64();
  for (int i = 0; i < N; i++) x = fma(x, y, 1e-12);
  t1 = clock64(); if (threadIdx.x == 0) out[0] = (double)(t1 - t0) / N;
  // DADD chain
  t0 = clock64();
  for (int i = 0; i < N; i++) x = x + 1e-12;
  t1 = clock64(); if (threadIdx.x == 0) out[1] = (double)(t1 - t0) / N;
  // shfl double chain
  t0 = clock64();
  for (int i = 0; i < N; i++) x += __shfl_xor_sync(0xffffffffu, x, 1);
  t1 = clock64(); if (threadIdx.x == 0) out[2] = (double)(t1 - t0) / N;
  // div chain
  t0 = clock64();
  for (int i = 0; i < N; i++) x = 1.0 / (x + 1.5);
  t1 = clock64(); if (threadIdx.x == 0) out[3] = (double)(t1 - t0) / N;
  // sqrt chain
  t0 = clock64();
  for (int i = 0; i < N; i++) x = sqrt(x + 1.5);
  t1 = clock64(); if (threadIdx.x == 0) out[4] = (double)(t1 - t0) / N;
  // rsqrt chain
  t0 = clock64();
  for (int i = 0; i < N; i++) x = rsqrt(x + 1.5);
  t1 = clock64(); if (threadIdx.x == 0) out[5] = (double)(t1 - t0) / N;
  // smem load chain
  __shared__ double s[64];
  if (threadIdx.x < 64) s[threadIdx.x] = threadIdx.x * 0;
  __syncwarp();
  int idx = threadIdx.x & 31;
  t0 = clock64();
  for (int i = 0; i < N; i++) { x += s[idx]; idx = (int)(s[idx]) + (threadIdx.x & 31); }
  t1 = clock64(); if (threadIdx.x == 0) out[6] = (double)(t1 - t0) / N;
  // syncthreads (1 warp)
  t0 = clock64();
  for (int i = 0; i < N; i++) { __syncthreads(); }
  t1 = clock64(); if (threadIdx.x == 0) out[7] = (double)(t1 - t0) / N;
  out[8 + threadIdx.x % 4] = x;
}
int main() {
  double* d; cudaMalloc(&d, 64 * 8);
  for (int threads : {32, 512}) {
    k<<<1, threads>>>(d, 1.0, 0); k<<<1, threads>>>(d, 1.0, 0);
    double h[8]; cudaMemcpy(h, d, 64, cudaMemcpyDeviceToHost);
    printf("threads %d: dfma %.1f dadd %.1f shfl(d) %.1f div %.1f sqrt %.1f rsqrt %.1f lds %.1f bar %.1f\n", threads,
           h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7]);
  }
  return 0;
}
