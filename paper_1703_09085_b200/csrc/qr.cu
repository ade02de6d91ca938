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
#include <cstdio>
#include <cstdlib>

#include "kernels.h"

namespace hm {

#ifdef HM_PHASE_TIMING
#define QT_INIT long long qt0 = clock64(), qt_panel = 0, qt_t = 0, qt_trail = 0
#define QT_MARK(acc)                        \
  do {                                      \
    __syncthreads();                        \
    const long long t_ = clock64();         \
    acc += t_ - qt0;                        \
    qt0 = t_;                               \
  } while (0)
#else
#define QT_INIT do {} while (0)
#define QT_MARK(acc) do {} while (0)
#endif

namespace {
constexpr int kNbMax = 16;

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// D(8x8) += A(8x4) B(4x8), FP64 tensor pipe (DMMA.8x8x4); fragments as in eval.cu
__device__ __forceinline__ void dmma_qr(double (&d)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d[0]), "+d"(d[1])
      : "d"(a), "d"(b));
}

}  // namespace

// Instantiated per launch shape (the body reads blockDim.x): <512, 1> for
// the 24 K-double buckets (one CTA per SM by shared memory), <256, 2> for
// 12 K, <256, 3> for 6 K -- register caps that let that many CTAs share an SM.
// kRB: trailing-update rows per lane in flight (x 2 columns).
template <int kThreads, int kMinBlocks, int kRB, bool kDmmaTrail>
__global__ void __launch_bounds__(kThreads, kMinBlocks) k_qr_blocked(const QrJob* __restrict__ jobs, int cap) {
  extern __shared__ double Vs[];            // panel / V (rows x nb), column-major
  __shared__ double T[kNbMax * kNbMax];     // upper triangular, column-major
  // (the DMMA variant needs more: G holds the -T^T W block (16 x 32), red2 the
  // W partials; the FFMA variants keep the smaller footprint -> more L1)
  __shared__ double G[kDmmaTrail ? 2 * kNbMax * kNbMax : kNbMax * kNbMax];   // V^T V
  __shared__ double red2[kDmmaTrail && kThreads >= 512 ? 4 * 16 * kNbMax : 2 * 16 * kNbMax];  // per-warp
                                            // partial sums (<= 16 warps), double-buffered
  __shared__ double piv[2 * kNbMax];        // pivot row of the current column, double-buffered
  __shared__ double stau[kNbMax];
  const QrJob J = jobs[blockIdx.x];
  const int m = J.m, n = J.n, lda = J.lda;
  double* A = J.A;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, NT = blockDim.x, NW = NT >> 5;
  int nb = kNbMax;
  while (nb > 1 && (int64_t)(m + (kDmmaTrail ? 15 : 0)) * nb > cap) nb >>= 1;
  QT_INIT;
  for (int k0 = 0; k0 < n; k0 += nb) {
    const int kb = min(nb, n - k0);
    const int rows = m - k0;
    // panel leading dimension = 4 (mod 16) for the DMMA trailing update
    // (conflict-free fragment loads); unpadded for the FFMA update
    const int ldp = kDmmaTrail ? rows + ((4 - (rows & 15)) & 15) : rows;
    // 1. load panel
    for (int64_t e = tid; e < (int64_t)rows * kb; e += NT) {
      const int i = (int)(e % rows), j = (int)(e / rows);
      Vs[i + (int64_t)j * ldp] = A[(k0 + i) + (int64_t)(k0 + j) * lda];
    }
    __syncthreads();
    // 2. unblocked Householder on the panel (in shared memory), ONE barrier per
    //    column: thread tid owns rows i = tid (mod NT) for the whole panel; one
    //    pass gives x.x and x.y_c for every later column c (x = column j below
    //    the diagonal); the pivot row j is published through piv[] by its
    //    owner; every thread then derives beta, tau and the column updates
    //    itself.  red / piv are double-buffered by the parity of j.
    for (int j = 0; j < kb; j++) {
      const int nc = kb - j;               // slot 0: x.x ; slot q: x.y_{j+q}
      const double* x = Vs + (int64_t)j * ldp;
      double part[kNbMax];
#pragma unroll
      for (int q = 0; q < kNbMax; q++) part[q] = 0.0;
      const int i0 = tid > j ? tid : tid + ((j - tid) / NT + 1) * NT;   // first owned row below j
      for (int i = i0; i < rows; i += NT) {
        const double xi = x[i];
#pragma unroll
        for (int q = 0; q < kNbMax; q++)
          if (q < nc) part[q] = fma(xi, Vs[i + (int64_t)(j + q) * ldp], part[q]);
      }
      double* rb = red2 + (j & 1) * (16 * kNbMax);
      double* pv = piv + (j & 1) * kNbMax;
      // warp reduce-scatter of the 16 slots (16 shuffles instead of 80): after
      // the xor-16/8/4/2 halvings lane L holds slot L >> 1 summed over its
      // half-warp partners, the xor-1 step completes it
      {
        double h8[8], h4[4], h2[2];
        const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4, b1 = lane & 2;
#pragma unroll
        for (int q = 0; q < 8; q++) {
          const double send = b4 ? part[q] : part[q + 8];
          h8[q] = (b4 ? part[q + 8] : part[q]) + __shfl_xor_sync(0xffffffffu, send, 16);
        }
#pragma unroll
        for (int q = 0; q < 4; q++) {
          const double send = b3 ? h8[q] : h8[q + 4];
          h4[q] = (b3 ? h8[q + 4] : h8[q]) + __shfl_xor_sync(0xffffffffu, send, 8);
        }
#pragma unroll
        for (int q = 0; q < 2; q++) {
          const double send = b2 ? h4[q] : h4[q + 2];
          h2[q] = (b2 ? h4[q + 2] : h4[q]) + __shfl_xor_sync(0xffffffffu, send, 4);
        }
        const double send = b1 ? h2[0] : h2[1];
        double h1 = (b1 ? h2[1] : h2[0]) + __shfl_xor_sync(0xffffffffu, send, 2);
        h1 += __shfl_xor_sync(0xffffffffu, h1, 1);
        const int slot = (b4 ? 8 : 0) + (b3 ? 4 : 0) + (b2 ? 2 : 0) + (b1 ? 1 : 0);
        if ((lane & 1) == 0 && slot < nc) rb[warp * kNbMax + slot] = h1;
      }
      if (tid == j % NT) {
#pragma unroll
        for (int q = 0; q < kNbMax; q++)
          if (q < nc) pv[q] = Vs[j + (int64_t)(j + q) * ldp];
      }
      __syncthreads();
      // lane q of every warp totals slot q over the warps (loads issued together)
      double tq = 0.0;
      if (lane < nc) {
        double r16[16];
#pragma unroll
        for (int w = 0; w < 16; w++) r16[w] = w < NW ? rb[w * kNbMax + lane] : 0.0;
#pragma unroll
        for (int w = 0; w < 16; w++) tq += r16[w];
      }
      const double xn2 = __shfl_sync(0xffffffffu, tq, 0);
      const double alpha = pv[0];
      double t = 0.0, sc = 0.0, beta = alpha;
      if (xn2 > 0.0) {
        beta = -copysign(sqrt(alpha * alpha + xn2), alpha);
        t = (beta - alpha) / beta;
        sc = 1.0 / (alpha - beta);
      }
      // d_q = tau (y_q[j] + v.y_q below), v = sc x below the pivot
      double dq = 0.0;
      if (lane >= 1 && lane < nc) dq = (pv[lane] + sc * tq) * t;
      double d[kNbMax];
#pragma unroll
      for (int q = 1; q < kNbMax; q++) d[q] = __shfl_sync(0xffffffffu, dq, q);
      if (tid == 0) { J.tau[k0 + j] = t; stau[j] = t; }
      if (tid == j % NT) {
        Vs[j + (int64_t)j * ldp] = beta;
#pragma unroll
        for (int q = 1; q < kNbMax; q++)
          if (q < nc) Vs[j + (int64_t)(j + q) * ldp] = pv[q] - d[q];
      }
      if (t != 0.0)
        for (int i = i0; i < rows; i += NT) {
          const double vi = Vs[i + (int64_t)j * ldp] * sc;
          Vs[i + (int64_t)j * ldp] = vi;
#pragma unroll
          for (int q = 1; q < kNbMax; q++)
            if (q < nc) Vs[i + (int64_t)(j + q) * ldp] -= d[q] * vi;
        }
    }
    __syncthreads();
    // 3. write the panel (R + reflectors) back; make V explicit (unit diagonal, zero above)
    for (int64_t e = tid; e < (int64_t)rows * kb; e += NT) {
      const int i = (int)(e % rows), j = (int)(e / rows);
      A[(k0 + i) + (int64_t)(k0 + j) * lda] = Vs[i + (int64_t)j * ldp];
    }
    __syncthreads();
    for (int64_t e = tid; e < (int64_t)kb * kb; e += NT) {
      const int i = (int)(e % kb), j = (int)(e / kb);
      if (i < j) Vs[i + (int64_t)j * ldp] = 0.0;
      else if (i == j) Vs[i + (int64_t)j * ldp] = 1.0;
    }
    __syncthreads();
    QT_MARK(qt_panel);
    const int ncol = n - k0 - kb;
    const bool wantT = J.T != nullptr && nb == kNbMax;   // panel factors for k_applyq
    if (ncol <= 0 && !wantT) continue;
    // 4. T (dlarft, forward columnwise): G = V^T V, T(i,i) = tau_i,
    //    T(0:i, i) = -tau_i T(0:i,0:i) G(0:i, i)
    for (int pr = warp; pr < kb * kb; pr += NW) {
      const int a = pr % kb, b = pr / kb;
      if (a >= b) continue;
      const double* va = Vs + (int64_t)a * ldp;
      const double* vb = Vs + (int64_t)b * ldp;
      double d = 0.0;
      for (int i = b + lane; i < rows; i += 32) d = fma(va[i], vb[i], d);   // va, vb zero above b
      d = wsum(d);
      if (lane == 0) G[a + b * kNbMax] = d;
    }
    __syncthreads();
    // lane r of warp 0 computes row r of T (it only needs its own row and G)
    if (warp == 0 && lane < kb) {
      const int r = lane;
      for (int i = r; i < kb; i++) {
        if (i == r) { T[r + r * kNbMax] = stau[r]; continue; }
        double s = 0.0;
        for (int q = r; q < i; q++) s = fma(T[r + q * kNbMax], G[q + i * kNbMax], s);
        T[r + i * kNbMax] = -stau[i] * s;
      }
    }
    __syncthreads();
    if (wantT)
      for (int e = tid; e < kNbMax * kNbMax; e += NT) J.T[(int64_t)(k0 / kNbMax) * kNbMax * kNbMax + e] = T[e];
    QT_MARK(qt_t);
    if (ncol <= 0) continue;
    if (kDmmaTrail) {
      // 5'. trailing update on the FP64 tensor pipe, 32 columns at a time:
      //     W = V^T A (warp t owns the 8x8 tile (qt, ct) of the 16 x 32 block, the
      //     two warp groups of a 512-thread CTA split the rows), Zn = -T^T W,
      //     A += V Zn (8-row tiles round-robin over the warps)
      double* Wp = red2;
      double* Zn = G;
      const int NWG = NW >> 3;
      const int lr = lane >> 2, lk = lane & 3;
      double* At = A + k0 + (int64_t)(k0 + kb) * lda;
      for (int cb = 0; cb < ncol; cb += 32) {
        const int wcb = min(32, ncol - cb);
        {
          const int t = warp & 7, g = warp >> 3;
          const int qt = t & 1, ct = t >> 1;
          const int q = qt * 8 + lr, jc = ct * 8 + lr;
          const bool qok = q < kb, cok = jc < wcb;
          const double* vq = Vs + (int64_t)q * ldp;
          const double* ac = At + (int64_t)(cb + (cok ? jc : 0)) * lda;
          double d[2] = {0.0, 0.0};
#pragma unroll 4
          for (int i0 = 4 * g; i0 < rows; i0 += 4 * NWG) {
            const int i = i0 + lk;
            const double a = (qok && i < rows) ? vq[i] : 0.0;
            const double b = (cok && i < rows) ? ac[i] : 0.0;
            dmma_qr(d, a, b);
          }
          if (g < NWG) {
            double* w = Wp + g * 512;
            w[q + (ct * 8 + 2 * lk) * 16] = d[0];
            w[q + (ct * 8 + 2 * lk + 1) * 16] = d[1];
          }
        }
        __syncthreads();
        for (int e = tid; e < 512; e += NT) {   // Zn(q, j) = -sum_{r <= q} T(r, q) W(r, j)
          const int q = e & 15, j = e >> 4;
          double sacc = 0.0;
          if (q < kb)
            for (int r = 0; r <= q; r++) {
              double wv = Wp[r + j * 16];
              if (NWG > 1) wv += Wp[512 + r + j * 16];
              sacc = fma(T[r + q * kNbMax], wv, sacc);
            }
          Zn[q + j * 16] = -sacc;
        }
        __syncthreads();
        {
          double bz[4][4];
#pragma unroll
          for (int ct = 0; ct < 4; ct++)
#pragma unroll
            for (int ks = 0; ks < 4; ks++) bz[ct][ks] = Zn[(ks * 4 + lk) + (ct * 8 + lr) * 16];
          const int nrt = (rows + 7) >> 3;
          for (int rt = warp; rt < nrt; rt += NW) {
            const int i = rt * 8 + lr;
            double a[4];
#pragma unroll
            for (int ks = 0; ks < 4; ks++) {
              const int q = ks * 4 + lk;
              a[ks] = (q < kb && i < rows) ? Vs[i + (int64_t)q * ldp] : 0.0;
            }
#pragma unroll
            for (int ct = 0; ct < 4; ct++) {
              if (ct * 8 >= wcb) break;   // warp-uniform
              double d[2];
#pragma unroll
              for (int h = 0; h < 2; h++) {
                const int j = ct * 8 + 2 * lk + h;
                d[h] = (i < rows && j < wcb) ? At[i + (int64_t)(cb + j) * lda] : 0.0;
              }
#pragma unroll
              for (int ks = 0; ks < 4; ks++) dmma_qr(d, a[ks], bz[ct][ks]);
#pragma unroll
              for (int h = 0; h < 2; h++) {
                const int j = ct * 8 + 2 * lk + h;
                if (i < rows && j < wcb) At[i + (int64_t)(cb + j) * lda] = d[h];
              }
            }
          }
        }
        __syncthreads();
      }
      QT_MARK(qt_trail);
      continue;
    }
    // 5. trailing update, one warp per PAIR of columns (each V element read
    //    from shared memory feeds two FMAs): a <- a - V (T^T (V^T a))
    for (int c2 = 2 * warp; c2 < ncol; c2 += 2 * NW) {
      double* a0 = A + k0 + (int64_t)(k0 + kb + c2) * lda;
      const bool two = c2 + 1 < ncol;
      double* a1 = two ? a0 + lda : a0;
      double w0[kNbMax], w1[kNbMax];
#pragma unroll
      for (int q = 0; q < kNbMax; q++) w0[q] = w1[q] = 0.0;
      // rows in blocks of kRB per lane: 2 kRB global loads in flight per lane
      int i = lane;
      for (; i + 32 * (kRB - 1) < rows; i += 32 * kRB) {
        double x0[kRB], x1[kRB];
#pragma unroll
        for (int u = 0; u < kRB; u++) { x0[u] = a0[i + 32 * u]; x1[u] = a1[i + 32 * u]; }
#pragma unroll
        for (int u = 0; u < kRB; u++)
#pragma unroll
          for (int q = 0; q < kNbMax; q++)
            if (q < kb) {
              const double v = Vs[i + 32 * u + q * ldp];
              w0[q] = fma(v, x0[u], w0[q]);
              w1[q] = fma(v, x1[u], w1[q]);
            }
      }
      for (; i < rows; i += 32) {
        const double x0 = a0[i], x1 = a1[i];
#pragma unroll
        for (int q = 0; q < kNbMax; q++)
          if (q < kb) {
            const double v = Vs[i + q * ldp];
            w0[q] = fma(v, x0, w0[q]);
            w1[q] = fma(v, x1, w1[q]);
          }
      }
#pragma unroll
      for (int q = 0; q < kNbMax; q++) { w0[q] = wsum(w0[q]); w1[q] = wsum(w1[q]); }
      // z = T^T w in place, from the last row up ((T^T w)_q = sum_{r<=q} T(r,q) w_r)
#pragma unroll
      for (int q = kNbMax - 1; q >= 0; q--) {
        double s0 = 0.0, s1 = 0.0;
#pragma unroll
        for (int r = 0; r <= q; r++)
          if (q < kb) {
            const double tr = T[r + q * kNbMax];
            s0 = fma(tr, w0[r], s0);
            s1 = fma(tr, w1[r], s1);
          }
        w0[q] = s0;
        w1[q] = s1;
      }
      i = lane;
      for (; i + 32 * (kRB - 1) < rows; i += 32 * kRB) {
        double x0[kRB], x1[kRB];
#pragma unroll
        for (int u = 0; u < kRB; u++) { x0[u] = a0[i + 32 * u]; x1[u] = a1[i + 32 * u]; }
#pragma unroll
        for (int u = 0; u < kRB; u++) {
          double s0 = 0.0, s1 = 0.0;
#pragma unroll
          for (int q = 0; q < kNbMax; q++)
            if (q < kb) {
              const double v = Vs[i + 32 * u + q * ldp];
              s0 = fma(v, w0[q], s0);
              s1 = fma(v, w1[q], s1);
            }
          x0[u] -= s0;
          x1[u] -= s1;
        }
#pragma unroll
        for (int u = 0; u < kRB; u++) {
          a0[i + 32 * u] = x0[u];
          if (two) a1[i + 32 * u] = x1[u];
        }
      }
      for (; i < rows; i += 32) {
        double s0 = 0.0, s1 = 0.0;
#pragma unroll
        for (int q = 0; q < kNbMax; q++)
          if (q < kb) {
            const double v = Vs[i + q * ldp];
            s0 = fma(v, w0[q], s0);
            s1 = fma(v, w1[q], s1);
          }
        a0[i] -= s0;
        if (two) a1[i] -= s1;
      }
    }
    __syncthreads();
    QT_MARK(qt_trail);
  }
#ifdef HM_PHASE_TIMING
  if (blockIdx.x == 0 && threadIdx.x == 0)
    printf("[qr] m=%d n=%d nb=%d panel %lld T %lld trailing %lld cycles\n", m, n, nb, qt_panel, qt_t, qt_trail);
#endif
}

// ---------------------------------------------------------------------------
// Stepped blocked QR: the same factorisation as k_qr_blocked
// (16-column panels, compact-WY T per panel, LAPACK layout), but the batch
// advances panel by panel with TWO kernels per step:
//   k_qrs_panel : one CTA per job factors the 16-column panel in shared memory
//                 (the Householder loop of k_qr_blocked) and writes R, the
//                 reflectors and the panel's T factor;
//   k_qrs_update: one CTA per (job, 32 trailing columns): W = V^T A_slab,
//                 Z = -T^T W, A_slab += V Z on the FP64 tensor pipe (DMMA),
//                 V read straight from the factored panel in global memory / L2.
// The trailing update -- 2 m l^2 of the 2 m l^2 QR flops -- is spread over the
// whole GPU instead of running inside the job's one CTA, and no CTA holds
// more than one panel in shared memory.
template <int kThreads, int kMinBlocks>
__global__ void __launch_bounds__(kThreads, kMinBlocks) k_qrs_panel(const QrJob* __restrict__ jobs, int k0) {
  extern __shared__ double Vs[];            // panel (rows x 16), column-major, ld = rows
  __shared__ double T[kNbMax * kNbMax];
  __shared__ double G[kNbMax * kNbMax];
  __shared__ double red2[2 * 16 * kNbMax];
  __shared__ double piv[2 * kNbMax];
  __shared__ double stau[kNbMax];
  const QrJob J = jobs[blockIdx.x];
  const int m = J.m, n = J.n, lda = J.lda;
  if (k0 >= n) return;
  double* A = J.A;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, NT = kThreads, NW = NT >> 5;
  const int kb = min(kNbMax, n - k0);
  const int rows = m - k0;
  const int ldp = rows;
  {
    const double* Ap = A + k0 + (int64_t)k0 * lda;
    for (int j = 0; j < kb; j++)
      for (int i = tid; i < rows; i += NT) Vs[i + (int64_t)j * ldp] = Ap[i + (int64_t)j * lda];
  }
  __syncthreads();
  for (int j = 0; j < kb; j++) {
    const int nc = kb - j;
    const double* x = Vs + (int64_t)j * ldp;
    double part[kNbMax];
#pragma unroll
    for (int q = 0; q < kNbMax; q++) part[q] = 0.0;
    const int i0 = tid > j ? tid : tid + ((j - tid) / NT + 1) * NT;
    for (int i = i0; i < rows; i += NT) {
      const double xi = x[i];
#pragma unroll
      for (int q = 0; q < kNbMax; q++)
        if (q < nc) part[q] = fma(xi, Vs[i + (int64_t)(j + q) * ldp], part[q]);
    }
    double* rb = red2 + (j & 1) * (16 * kNbMax);
    double* pv = piv + (j & 1) * kNbMax;
    {
      double h8[8], h4[4], h2[2];
      const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4, b1 = lane & 2;
#pragma unroll
      for (int q = 0; q < 8; q++) {
        const double send = b4 ? part[q] : part[q + 8];
        h8[q] = (b4 ? part[q + 8] : part[q]) + __shfl_xor_sync(0xffffffffu, send, 16);
      }
#pragma unroll
      for (int q = 0; q < 4; q++) {
        const double send = b3 ? h8[q] : h8[q + 4];
        h4[q] = (b3 ? h8[q + 4] : h8[q]) + __shfl_xor_sync(0xffffffffu, send, 8);
      }
#pragma unroll
      for (int q = 0; q < 2; q++) {
        const double send = b2 ? h4[q] : h4[q + 2];
        h2[q] = (b2 ? h4[q + 2] : h4[q]) + __shfl_xor_sync(0xffffffffu, send, 4);
      }
      const double send = b1 ? h2[0] : h2[1];
      double h1 = (b1 ? h2[1] : h2[0]) + __shfl_xor_sync(0xffffffffu, send, 2);
      h1 += __shfl_xor_sync(0xffffffffu, h1, 1);
      const int slot = (b4 ? 8 : 0) + (b3 ? 4 : 0) + (b2 ? 2 : 0) + (b1 ? 1 : 0);
      if ((lane & 1) == 0 && slot < nc) rb[warp * kNbMax + slot] = h1;
    }
    if (tid == j % NT) {
#pragma unroll
      for (int q = 0; q < kNbMax; q++)
        if (q < nc) pv[q] = Vs[j + (int64_t)(j + q) * ldp];
    }
    __syncthreads();
    double tq = 0.0;
    if (lane < nc) {
      double r16[16];
#pragma unroll
      for (int w = 0; w < 16; w++) r16[w] = w < NW ? rb[w * kNbMax + lane] : 0.0;
#pragma unroll
      for (int w = 0; w < 16; w++) tq += r16[w];
    }
    const double xn2 = __shfl_sync(0xffffffffu, tq, 0);
    const double alpha = pv[0];
    double t = 0.0, sc = 0.0, beta = alpha;
    if (xn2 > 0.0) {
      beta = -copysign(sqrt(alpha * alpha + xn2), alpha);
      t = (beta - alpha) / beta;
      sc = 1.0 / (alpha - beta);
    }
    double dq = 0.0;
    if (lane >= 1 && lane < nc) dq = (pv[lane] + sc * tq) * t;
    double d[kNbMax];
#pragma unroll
    for (int q = 1; q < kNbMax; q++) d[q] = __shfl_sync(0xffffffffu, dq, q);
    if (tid == 0) { J.tau[k0 + j] = t; stau[j] = t; }
    if (tid == j % NT) {
      Vs[j + (int64_t)j * ldp] = beta;
#pragma unroll
      for (int q = 1; q < kNbMax; q++)
        if (q < nc) Vs[j + (int64_t)(j + q) * ldp] = pv[q] - d[q];
    }
    if (t != 0.0)
      for (int i = i0; i < rows; i += NT) {
        const double vi = Vs[i + (int64_t)j * ldp] * sc;
        Vs[i + (int64_t)j * ldp] = vi;
#pragma unroll
        for (int q = 1; q < kNbMax; q++)
          if (q < nc) Vs[i + (int64_t)(j + q) * ldp] -= d[q] * vi;
      }
  }
  __syncthreads();
  {
    double* Ap = A + k0 + (int64_t)k0 * lda;
    for (int j = 0; j < kb; j++)
      for (int i = tid; i < rows; i += NT) Ap[i + (int64_t)j * lda] = Vs[i + (int64_t)j * ldp];
  }
  __syncthreads();
  for (int e = tid; e < kb * kb; e += NT) {
    const int i = e % kb, j = e / kb;
    if (i < j) Vs[i + (int64_t)j * ldp] = 0.0;
    else if (i == j) Vs[i + (int64_t)j * ldp] = 1.0;
  }
  __syncthreads();
  // T (dlarft, forward columnwise) as in k_qr_blocked
  for (int pr = warp; pr < kb * kb; pr += NW) {
    const int a = pr % kb, b = pr / kb;
    if (a >= b) continue;
    const double* va = Vs + (int64_t)a * ldp;
    const double* vb = Vs + (int64_t)b * ldp;
    double d = 0.0;
    for (int i = b + lane; i < rows; i += 32) d = fma(va[i], vb[i], d);
    d = wsum(d);
    if (lane == 0) G[a + b * kNbMax] = d;
  }
  __syncthreads();
  if (warp == 0 && lane < kb) {
    const int r = lane;
    for (int i = r; i < kb; i++) {
      if (i == r) { T[r + r * kNbMax] = stau[r]; continue; }
      double s = 0.0;
      for (int q = r; q < i; q++) s = fma(T[r + q * kNbMax], G[q + i * kNbMax], s);
      T[r + i * kNbMax] = -stau[i] * s;
    }
  }
  __syncthreads();
  for (int e = tid; e < kNbMax * kNbMax; e += NT) {
    const int r = e & 15, q = e >> 4;
    J.T[(int64_t)(k0 / kNbMax) * kNbMax * kNbMax + e] = (r <= q && q < kb) ? T[e] : 0.0;
  }
}

// Trailing update of step k0 for 32 trailing columns of one job (blockIdx.y =
// job, blockIdx.x = column slab).  256 threads = 8 warps; rows are dealt to
// the warps 4 (phase 1) / 8 (phase 2) at a time.
__global__ void __launch_bounds__(256, 3) k_qrs_update(const QrJob* __restrict__ jobs, int k0) {
  __shared__ double Wp[8 * 512];   // per-warp partial W (16 x 32), then W itself in Wp[0..512)
  __shared__ double Zn[512];       // -T^T W (16 x 32)
  __shared__ double Ts[256];
  const QrJob J = jobs[blockIdx.y];
  const int n = J.n;
  if (k0 >= n) return;
  const int kb = min(kNbMax, n - k0);
  const int ncol = n - k0 - kb;
  const int cb = blockIdx.x * 32;
  if (cb >= ncol) return;
  const int wcb = min(32, ncol - cb);
  const int lda = J.lda, rows = J.m - k0;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int lr = lane >> 2, lk = lane & 3;
  const double* Vg = J.A + k0 + (int64_t)k0 * lda;            // panel: v(i, q), implicit unit diagonal
  double* At = J.A + k0 + (int64_t)(k0 + kb + cb) * lda;      // slab (rows x wcb)
  Ts[tid] = J.T[(int64_t)(k0 / kNbMax) * 256 + tid];
  // ---- phase 1: partial W = V^T A over this warp's rows
  double d[2][4][2];
#pragma unroll
  for (int a = 0; a < 2; a++)
#pragma unroll
    for (int b = 0; b < 4; b++) d[a][b][0] = d[a][b][1] = 0.0;
  const double* vq0 = Vg + (int64_t)min(lr, kb - 1) * lda;
  const double* vq1 = Vg + (int64_t)min(8 + lr, kb - 1) * lda;
  const bool q0ok = lr < kb, q1ok = 8 + lr < kb;
  const double* ac[4];
  bool cok[4];
#pragma unroll
  for (int ct = 0; ct < 4; ct++) {
    const int jc = ct * 8 + lr;
    cok[ct] = jc < wcb;
    ac[ct] = At + (int64_t)(cok[ct] ? jc : 0) * lda;
  }
  // the first 16 rows carry the unit triangle of V: masked loads
  for (int i0 = 4 * warp; i0 < rows; i0 += 32) {
    const int i = i0 + lk;
    const bool iok = i < rows;
    double a0 = 0.0, a1 = 0.0;
    if (i0 >= kNbMax) {
      if (iok) { a0 = q0ok ? vq0[i] : 0.0; a1 = q1ok ? vq1[i] : 0.0; }
    } else if (iok) {
      const int qa = lr, qb = 8 + lr;
      a0 = !q0ok ? 0.0 : (i > qa ? vq0[i] : (i == qa ? 1.0 : 0.0));
      a1 = !q1ok ? 0.0 : (i > qb ? vq1[i] : (i == qb ? 1.0 : 0.0));
    }
    double b[4];
#pragma unroll
    for (int ct = 0; ct < 4; ct++) b[ct] = (iok && cok[ct]) ? ac[ct][i] : 0.0;
#pragma unroll
    for (int ct = 0; ct < 4; ct++) {
      dmma_qr(d[0][ct], a0, b[ct]);
      dmma_qr(d[1][ct], a1, b[ct]);
    }
  }
  {
    double* w = Wp + warp * 512;
#pragma unroll
    for (int qt = 0; qt < 2; qt++)
#pragma unroll
      for (int ct = 0; ct < 4; ct++) {
        const int q = qt * 8 + lr;
        w[q + (ct * 8 + 2 * lk) * 16] = d[qt][ct][0];
        w[q + (ct * 8 + 2 * lk + 1) * 16] = d[qt][ct][1];
      }
  }
  __syncthreads();
  for (int e = tid; e < 512; e += 256) {
    double sacc = 0.0;
#pragma unroll
    for (int w = 0; w < 8; w++) sacc += Wp[w * 512 + e];
    Zn[e] = sacc;   // W, staged in Zn
  }
  __syncthreads();
  for (int e = tid; e < 512; e += 256) {   // Z(q, j) = -sum_{r <= q} T(r, q) W(r, j)
    const int q = e & 15, j = e >> 4;
    double sacc = 0.0;
    if (q < kb)
      for (int r = 0; r <= q; r++) sacc = fma(Ts[r + q * kNbMax], Zn[r + j * 16], sacc);
    Wp[e] = -sacc;
  }
  __syncthreads();
  // ---- phase 2: A_slab += V Z, 8-row tiles round-robin over the warps
  {
    double bz[4][4];
#pragma unroll
    for (int ct = 0; ct < 4; ct++)
#pragma unroll
      for (int ks = 0; ks < 4; ks++) bz[ct][ks] = Wp[(ks * 4 + lk) + (ct * 8 + lr) * 16];
    const int nrt = (rows + 7) >> 3;
    for (int rt = warp; rt < nrt; rt += 8) {
      const int i = rt * 8 + lr;
      const bool iok = i < rows;
      double a[4];
#pragma unroll
      for (int ks = 0; ks < 4; ks++) {
        const int q = ks * 4 + lk;
        double v = 0.0;
        if (q < kb && iok) v = (rt >= 2 || i > q) ? Vg[i + (int64_t)q * lda] : (i == q ? 1.0 : 0.0);
        a[ks] = v;
      }
      double c2[4][2];
#pragma unroll
      for (int ct = 0; ct < 4; ct++)
#pragma unroll
        for (int h = 0; h < 2; h++) {
          const int j = ct * 8 + 2 * lk + h;
          c2[ct][h] = (iok && j < wcb) ? At[i + (int64_t)j * lda] : 0.0;
        }
#pragma unroll
      for (int ct = 0; ct < 4; ct++)
#pragma unroll
        for (int ks = 0; ks < 4; ks++) dmma_qr(c2[ct], a[ks], bz[ct][ks]);
#pragma unroll
      for (int ct = 0; ct < 4; ct++)
#pragma unroll
        for (int h = 0; h < 2; h++) {
          const int j = ct * 8 + 2 * lk + h;
          if (iok && j < wcb) At[i + (int64_t)j * lda] = c2[ct][h];
        }
    }
  }
}

// jobs sorted by n (columns) descending; ncols[i] = n of job i (host copy).
// All jobs need m * 16 <= 24 K doubles and a T buffer.
void launch_qr_stepped(const QrJob* d_jobs, const int* ncols, int njobs, int max_m, cudaStream_t st) {
  if (njobs <= 0) return;
  const size_t smem = (size_t)max_m * kNbMax * sizeof(double);
  const bool big = max_m > 768;
  if (big) ensure_smem_attr((const void*)k_qrs_panel<512, 1>, 24 * 1024 * 8);
  else ensure_smem_attr((const void*)k_qrs_panel<256, 2>, 12 * 1024 * 8);
  int active = njobs;
  for (int k0 = 0; k0 < ncols[0]; k0 += kNbMax) {
    while (active > 0 && ncols[active - 1] <= k0) active--;
    if (active == 0) break;
    count_launch();
    if (big) k_qrs_panel<512, 1><<<active, 512, smem, st>>>(d_jobs, k0);
    else k_qrs_panel<256, 2><<<active, 256, smem, st>>>(d_jobs, k0);
    const int ncol = ncols[0] - k0 - kNbMax;
    if (ncol > 0) {
      int act2 = active;
      while (act2 > 0 && ncols[act2 - 1] <= k0 + kNbMax) act2--;
      if (act2 > 0) {
        count_launch();
        k_qrs_update<<<dim3((ncol + 31) / 32, act2), 256, 0, st>>>(d_jobs, k0);
      }
    }
  }
}

template <int kThreads, int kMinBlocks>
static void launch_qr_variant(const QrJob* d_jobs, int njobs, int cap, int rb, cudaStream_t st) {
  static const int dm = [] { const char* e = std::getenv("HM_QR_DMMA"); return e ? std::atoi(e) : 1; }();
  const bool use_dmma = dm && kThreads == 256 && cap <= 6 * 1024;
  // +256 doubles: the DMMA variant pads the panel leading dimension to 4 (mod 16)
  const int capx = cap + (use_dmma ? 256 : 0);
  {
    const int bytes = ((kThreads == 512 ? 24 : (kMinBlocks == 2 ? 12 : 6)) * 1024 + 256) * 8;
    ensure_smem_attr((const void*)k_qr_blocked<kThreads, kMinBlocks, 4, true>, bytes);
    ensure_smem_attr((const void*)k_qr_blocked<kThreads, kMinBlocks, 4, false>, bytes);
    ensure_smem_attr((const void*)k_qr_blocked<kThreads, kMinBlocks, 8, false>, bytes);
  }
  // DMMA trailing update: measured faster only for the 384-row bucket with
  // 256 threads (133 -> 115 ms per cfg-4 product); 768 rows +4 %, 1536 rows and
  // the 512-thread latency mode (one dependent DMMA chain per warp over all
  // rows) slower -- the FFMA column-pair update stays there
  if (use_dmma) k_qr_blocked<kThreads, kMinBlocks, 4, true><<<njobs, kThreads, (size_t)capx * 8, st>>>(d_jobs, capx);
  else if (rb == 8) k_qr_blocked<kThreads, kMinBlocks, 8, false><<<njobs, kThreads, (size_t)capx * 8, st>>>(d_jobs, capx);
  else k_qr_blocked<kThreads, kMinBlocks, 4, false><<<njobs, kThreads, (size_t)capx * 8, st>>>(d_jobs, capx);
}

void launch_qr_blocked(const QrJob* d_jobs, int njobs, int cap, cudaStream_t st) {
  if (njobs <= 0) return;
  if (cap > 24 * 1024) cap = 24 * 1024;
  count_launch();
  // <256, 3> (80 registers) spills ~650 B per thread: measured slower on B200
  // (6 K bucket 133 -> 177 ms per cfg-4 product), so off unless HM_QR_OCC3=1
  static const int occ3 = [] { const char* e = std::getenv("HM_QR_OCC3"); return e ? std::atoi(e) : 0; }();
  static const int rb = [] { const char* e = std::getenv("HM_QR_RB"); return e ? std::atoi(e) : 4; }();
  // <= 12 K doubles (96 KB): 256 threads, two CTAs per SM (measured on B200:
  // the 768-row bucket 194 -> 165 ms per cfg-4 product vs one 512-thread CTA)
  // fewer jobs than SMs (latency-bound, e.g. the H-LR critical path): 512
  // threads per QR whatever the bucket
  static const int lat = [] { const char* e = std::getenv("HM_QR_LAT512"); return e ? std::atoi(e) : 1; }();
  if (lat && njobs < 148) launch_qr_variant<512, 1>(d_jobs, njobs, cap, rb, st);
  else if (cap <= 6 * 1024 && occ3) launch_qr_variant<256, 3>(d_jobs, njobs, cap, rb, st);
  else if (cap <= 12 * 1024) launch_qr_variant<256, 2>(d_jobs, njobs, cap, rb, st);
  else launch_qr_variant<512, 1>(d_jobs, njobs, cap, rb, st);
}

}  // namespace hm
