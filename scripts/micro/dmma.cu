// Micro-benchmark: DMMA.8x8x4 (mma.sync m8n8k4 f64) dependent-chain latency and
// throughput with 1..8 independent accumulators, 1..16 warps per SM.  Diagnostics only.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}
template <int NACC>
__global__ void k(double* out, double seed, long long* cyc) {
  double d[NACC][2];
  for (int i = 0; i < NACC; i++) d[i][0] = d[i][1] = 0.0;
  const double a = seed + threadIdx.x * 1e-9, b = 1.0000001;
  const int N = 512;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < N; i++) {
#pragma unroll
    for (int j = 0; j < NACC; j++) dmma(d[j], a, b);
  }
  long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < NACC; i++) s += d[i][0] + d[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
template <int NACC>
void run(int threads, int blocks, double* d, long long* c) {
  k<NACC><<<blocks, threads>>>(d, 1.0, c); k<NACC><<<blocks, threads>>>(d, 1.0, c);
  long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("acc %d threads %4d blocks %3d: %.1f cycles per DMMA-round, %.2f cycles per DMMA per warp\n", NACC, threads, blocks, h / 512.0, h / 512.0 / NACC);
}
int main() {
  double* d; cudaMalloc(&d, 148 * 1024 * 8); long long* c; cudaMalloc(&c, 8);
  for (int th : {32, 128, 256, 512}) { run<1>(th, 1, d, c); run<2>(th, 1, d, c); run<4>(th, 1, d, c); run<8>(th, 1, d, c); }
  run<4>(256, 148, d, c); run<8>(512, 148, d, c);
  return 0;
}
