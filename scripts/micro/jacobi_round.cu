// Micro-benchmark: cycles per Jacobi round for c = 64 columns, one CTA.
// Variants isolate the cost of the rotation-parameter chain, the V update and
// the barrier.  Diagnostics only (not part of libhm).
#include <cstdio>
#include <cuda_runtime.h>

template <int G, int E, int MODE>
__global__ void k(double* out, int c, int rounds) {
  extern __shared__ double sm[];
  double* X = sm;
  double* V = sm + 64 * 65;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, NW = blockDim.x >> 5;
  constexpr int gpw = 32 / G;
  const int gl = lane & (G - 1);
  const int ldx = 65;
  for (int e = tid; e < 64 * 65; e += blockDim.x) { X[e] = 1.0 / (1 + e % 97) + (e % 13) * 1e-3; V[e] = (e % 66 == 0); }
  __syncthreads();
  const int cp = c;
  long long t0 = clock64();
  double acc = 0;
  for (int r = 0; r < rounds; r++) {
    const int rr = r % (cp - 1);
    for (int base = warp * gpw; base < (cp >> 1); base += NW * gpw) {
      const int pr = base + lane / G;
      int a = 0, b = 0;
      bool act = pr < (cp >> 1);
      if (act) {
        int x1 = pr - 1 + rr; if (x1 >= cp - 1) x1 -= cp - 1;
        a = pr == 0 ? 0 : x1 + 1;
        const int k2 = cp - 1 - pr;
        int x2 = k2 - 1 + rr; if (x2 >= cp - 1) x2 -= cp - 1;
        b = x2 + 1;
      }
      double* x = X + a * ldx + gl;
      double* y = X + b * ldx + gl;
      double xr[E], yr[E];
      double al = 0, be = 0, ga = 0;
#pragma unroll
      for (int u = 0; u < E; u++) { xr[u] = x[u * G]; yr[u] = y[u * G]; }
#pragma unroll
      for (int u = 0; u < E; u++) { al = fma(xr[u], xr[u], al); be = fma(yr[u], yr[u], be); ga = fma(xr[u], yr[u], ga); }
#pragma unroll
      for (int o = G >> 1; o > 0; o >>= 1) {
        al += __shfl_xor_sync(0xffffffffu, al, o);
        be += __shfl_xor_sync(0xffffffffu, be, o);
        ga += __shfl_xor_sync(0xffffffffu, ga, o);
      }
      double cs = 0.99995, sn = 0.0099;
      if (MODE == 4) {
        // rsqrt formulation with power-of-two scaling
        const double d0 = be - al, g0 = 2.0 * ga;
        const int ex = (max(__double2hiint(d0) & 0x7ff00000, __double2hiint(g0) & 0x7ff00000));
        const double scl = __hiloint2double(0x7fe00000 - ex, 0);   // ~ 2^-(e)
        const double d = d0 * scl, g = g0 * scl;
        const double rh = rsqrt(fma(d, d, g * g));
        const double c2 = fabs(d) * rh, s2 = fabs(g) * rh;
        const double hc = fma(0.5, c2, 0.5);
        const double r2 = rsqrt(hc);
        cs = hc * r2;
        sn = copysign(0.5 * s2 * r2, d * g) * 1e-3;
      } else if (MODE != 1) {
        const double d0 = be - al, g0 = 2.0 * ga;
        const double sc = 1.0 / fmax(fabs(d0), fabs(g0));
        const double d = d0 * sc, g = g0 * sc;
        const double tt = copysign(fabs(g) / (fabs(d) + sqrt(fma(d, d, g * g))), d * g);
        cs = rsqrt(fma(tt, tt, 1.0)); sn = cs * tt * 1e-3;
      }
      if (act) {
#pragma unroll
        for (int u = 0; u < E; u++) { x[u * G] = cs * xr[u] - sn * yr[u]; y[u * G] = sn * xr[u] + cs * yr[u]; }
        if (MODE != 2) {
          double* uu = V + a * ldx + gl;
          double* ww = V + b * ldx + gl;
#pragma unroll
          for (int u = 0; u < E; u++) { xr[u] = uu[u * G]; yr[u] = ww[u * G]; }
#pragma unroll
          for (int u = 0; u < E; u++) { uu[u * G] = cs * xr[u] - sn * yr[u]; ww[u * G] = sn * xr[u] + cs * yr[u]; }
        }
      }
      acc += al;
    }
    if (MODE != 3) __syncthreads(); else __syncwarp();
  }
  long long t1 = clock64();
  if (tid == 0) { out[0] = (double)(t1 - t0) / rounds; out[1] = acc; }
}

template <int G, int E, int MODE>
void run(const char* name, int threads) {
  double* d; cudaMalloc(&d, 16);
  cudaFuncSetAttribute(k<G, E, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 64 * 65 * 8);
  k<G, E, MODE><<<1, threads, 2 * 64 * 65 * 8>>>(d, 64, 630);
  k<G, E, MODE><<<1, threads, 2 * 64 * 65 * 8>>>(d, 64, 630);
  double h[2]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("%-28s G=%2d E=%d threads=%d: %.0f cycles/round\n", name, G, E, threads, h[0]);
  cudaFree(d);
}

int main() {
  run<8, 8, 0>("full", 256);
  run<16, 4, 0>("full", 512);
  run<32, 2, 0>("full", 1024);
  run<16, 4, 1>("no params", 512);
  run<16, 4, 2>("no V", 512);
  run<16, 4, 3>("no barrier", 512);
  run<8, 8, 1>("no params", 256);
  run<8, 8, 3>("no barrier", 256);
  run<16, 4, 4>("rsqrt params", 512);
  run<8, 8, 4>("rsqrt params", 256);
  return 0;
}
