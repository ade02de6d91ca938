// Blocked Householder QR (LAPACK dgeqrf layout: R in the upper triangle,
// reflectors below, tau) of tall stacked factors A (m x n, m > n) that do not
// fit in shared memory -- the QR of the TRUNC stacks (§3
// "Truncation"; Fig. 2 "Find thin QR factorization").
//
// One CTA per panel matrix.  Panels of nb columns (nb*rows fit in shared
// memory) are factorized in shared memory; the trailing columns are updated
// with the compact-WY form Q^T = I - V T^T V^T (dlarft / dlarfb), i.e. two
// streaming passes over the trailing matrix per panel instead of nb passes.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "kernels.h"

namespace hm {

namespace {
constexpr int kNbMax = 16;

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ double bsum(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = wsum(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    double s = (lane < nw) ? red[lane] : 0.0;
    s = wsum(s);
    if (lane == 0) red[0] = s;
  }
  __syncthreads();
  const double s = red[0];
  __syncthreads();
  return s;
}
}  // namespace

__global__ void k_qr_blocked(const QrJob* __restrict__ jobs, int cap) {
  extern __shared__ double Vs[];            // panel / V (rows x nb), column-major
  __shared__ double red[32];
  __shared__ double T[kNbMax * kNbMax];     // upper triangular, column-major
  __shared__ double G[kNbMax * kNbMax];     // V^T V
  __shared__ double s_tau, s_scale;
  const QrJob J = jobs[blockIdx.x];
  const int m = J.m, n = J.n, lda = J.lda;
  double* A = J.A;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, NT = blockDim.x, NW = NT >> 5;
  int nb = kNbMax;
  while (nb > 1 && (int64_t)m * nb > cap) nb >>= 1;
  for (int k0 = 0; k0 < n; k0 += nb) {
    const int kb = min(nb, n - k0);
    const int rows = m - k0;
    // 1. load panel
    for (int64_t e = tid; e < (int64_t)rows * kb; e += NT) {
      const int i = (int)(e % rows), j = (int)(e / rows);
      Vs[e] = A[(k0 + i) + (int64_t)(k0 + j) * lda];
    }
    __syncthreads();
    // 2. unblocked Householder on the panel (in shared memory)
    for (int j = 0; j < kb; j++) {
      double* x = Vs + (int64_t)j * rows;
      double pp = 0.0;
      for (int i = j + 1 + tid; i < rows; i += NT) pp = fma(x[i], x[i], pp);
      const double xn2 = bsum(pp, red);
      if (tid == 0) {
        const double alpha = x[j];
        double t = 0.0, sc = 0.0, beta = alpha;
        if (xn2 > 0.0) {
          beta = -copysign(sqrt(alpha * alpha + xn2), alpha);
          t = (beta - alpha) / beta;
          sc = 1.0 / (alpha - beta);
        }
        x[j] = beta;
        J.tau[k0 + j] = t;
        s_tau = t;
        s_scale = sc;
      }
      __syncthreads();
      const double t = s_tau, sc = s_scale;
      if (t != 0.0)
        for (int i = j + 1 + tid; i < rows; i += NT) x[i] *= sc;
      __syncthreads();
      if (t != 0.0) {
        for (int c = j + 1 + warp; c < kb; c += NW) {
          double* y = Vs + (int64_t)c * rows;
          double d = 0.0;
          for (int i = j + 1 + lane; i < rows; i += 32) d = fma(x[i], y[i], d);
          d = (wsum(d) + y[j]) * t;
          if (lane == 0) y[j] -= d;
          for (int i = j + 1 + lane; i < rows; i += 32) y[i] -= d * x[i];
        }
      }
      __syncthreads();
    }
    // 3. write the panel (R + reflectors) back; make V explicit (unit diagonal, zero above)
    for (int64_t e = tid; e < (int64_t)rows * kb; e += NT) {
      const int i = (int)(e % rows), j = (int)(e / rows);
      A[(k0 + i) + (int64_t)(k0 + j) * lda] = Vs[e];
    }
    __syncthreads();
    for (int64_t e = tid; e < (int64_t)kb * kb; e += NT) {
      const int i = (int)(e % kb), j = (int)(e / kb);
      if (i < j) Vs[i + (int64_t)j * rows] = 0.0;
      else if (i == j) Vs[i + (int64_t)j * rows] = 1.0;
    }
    __syncthreads();
    const int ncol = n - k0 - kb;
    if (ncol <= 0) continue;
    // 4. T (dlarft, forward columnwise): G = V^T V, T(i,i) = tau_i,
    //    T(0:i, i) = -tau_i T(0:i,0:i) G(0:i, i)
    for (int pr = warp; pr < kb * kb; pr += NW) {
      const int a = pr % kb, b = pr / kb;
      if (a >= b) continue;
      const double* va = Vs + (int64_t)a * rows;
      const double* vb = Vs + (int64_t)b * rows;
      double d = 0.0;
      for (int i = b + lane; i < rows; i += 32) d = fma(va[i], vb[i], d);   // va, vb zero above b
      d = wsum(d);
      if (lane == 0) G[a + b * kNbMax] = d;
    }
    __syncthreads();
    if (tid == 0) {
      for (int i = 0; i < kb; i++) {
        const double ti = J.tau[k0 + i];
        for (int r = 0; r < i; r++) {
          double s = 0.0;
          for (int q = r; q < i; q++) s += T[r + q * kNbMax] * G[q + i * kNbMax];
          T[r + i * kNbMax] = -ti * s;
        }
        T[i + i * kNbMax] = ti;
      }
    }
    __syncthreads();
    // 5. trailing update, one warp per column: a <- a - V (T^T (V^T a))
    for (int cc = warp; cc < ncol; cc += NW) {
      double* a = A + k0 + (int64_t)(k0 + kb + cc) * lda;
      double w[kNbMax];
#pragma unroll
      for (int q = 0; q < kNbMax; q++) w[q] = 0.0;
      for (int i = lane; i < rows; i += 32) {
        const double ai = a[i];
#pragma unroll
        for (int q = 0; q < kNbMax; q++)
          if (q < kb) w[q] = fma(Vs[i + (int64_t)q * rows], ai, w[q]);
      }
#pragma unroll
      for (int q = 0; q < kNbMax; q++) w[q] = wsum(w[q]);
      double z[kNbMax];
#pragma unroll
      for (int q = 0; q < kNbMax; q++) {
        double s = 0.0;
#pragma unroll
        for (int r = 0; r < kNbMax; r++)
          if (r <= q && q < kb) s = fma(T[r + q * kNbMax], w[r], s);   // (T^T w)_q = sum_{r<=q} T(r,q) w_r
        z[q] = s;
      }
      for (int i = lane; i < rows; i += 32) {
        double s = 0.0;
#pragma unroll
        for (int q = 0; q < kNbMax; q++)
          if (q < kb) s = fma(Vs[i + (int64_t)q * rows], z[q], s);
        a[i] -= s;
      }
    }
    __syncthreads();
  }
}

void launch_qr_blocked(const QrJob* d_jobs, int njobs, int cap, cudaStream_t st) {
  if (njobs <= 0) return;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_qr_blocked, cudaFuncAttributeMaxDynamicSharedMemorySize, 24 * 1024 * 8);
    attr = true;
  }
  if (cap > 24 * 1024) cap = 24 * 1024;
  count_launch();
  k_qr_blocked<<<njobs, cap <= 6 * 1024 ? 256 : 512, (size_t)cap * 8, st>>>(d_jobs, cap);
}

}  // namespace hm
