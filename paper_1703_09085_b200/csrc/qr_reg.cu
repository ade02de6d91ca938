// Blocked Householder QR with a REGISTER-resident panel (LAPACK dgeqrf layout,
// compact-WY T per 16-column panel; same factorisation as k_qr_blocked in
// qr.cu) for the stacked TRUNC factors of up to 768 rows (§3
// "Truncation"; Fig. 2 "Find thin QR factorization").
//
// One CTA of kNT threads per matrix.  Thread tid owns the panel rows
// tid + kNT u (u < kRPT) and keeps their 16 panel entries in registers for the
// whole panel factorisation: a Householder column step is register FMAs, one
// warp reduce-scatter, ONE barrier and a 16-value broadcast -- no pass over
// shared memory (k_qr_blocked: two shared-memory passes and ~750 instructions
// per warp and column, measured 5 K cycles per column at 256 and 512 threads).
// The trailing update runs on the FP64 tensor pipe (DMMA.8x8x4): W = V^T A
// (warp w owns 8 trailing columns, no cross-warp reduction), Z = -T^T W in
// place, A += V Z (8-row tiles round-robin over the warps), V staged in shared
// memory with a leading dimension = 4 (mod 16) (conflict-free fragments), the
// trailing matrix read straight from global memory / L2.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <cstdio>
#include <cstdlib>

#include "kernels.h"

namespace hm {

namespace {
constexpr int kNb = 16;

__device__ __forceinline__ void dmma_r(double (&d)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d[0]), "+d"(d[1])
      : "d"(a), "d"(b));
}

__device__ __forceinline__ void prefetch_l1(const void* p) { asm volatile("prefetch.global.L1 [%0];" ::"l"(p)); }

__host__ __device__ __forceinline__ int ld4mod16(int n) { return n + ((4 - (n & 15)) & 15); }
}  // namespace

#ifdef HM_PHASE_TIMING
#define RT_INIT long long rt0 = clock64(), rt_panel = 0, rt_t = 0, rt_trail = 0
#define RT_MARK(acc)                        \
  do {                                      \
    __syncthreads();                        \
    const long long t_ = clock64();         \
    acc += t_ - rt0;                        \
    rt0 = t_;                               \
  } while (0)
#else
#define RT_INIT do {} while (0)
#define RT_MARK(acc) do {} while (0)
#endif

template <int kNT, int kRPT, int kMinBlocks>
__global__ void __launch_bounds__(kNT, kMinBlocks) k_qr_reg(const QrJob* __restrict__ jobs) {
  constexpr int NW = kNT / 32;
  constexpr int CB = 8 * NW;                 // trailing columns per block (8 per warp)
  extern __shared__ double smq[];
  __shared__ double T[kNb * kNb];            // upper triangular, column-major, zero elsewhere
  __shared__ double red[2 * NW * kNb];       // per-warp partial dots, double-buffered
  __shared__ double piv[2 * kNb];            // pivot row, double-buffered
  __shared__ double stau[kNb];
  const QrJob J = jobs[blockIdx.x];
  const int m = J.m, n = J.n, lda = J.lda;
  double* const A = J.A;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int lr = lane >> 2, lk = lane & 3;
  const int ldp = ld4mod16(m);
  double* Vs = smq;                          // ldp x 16: explicit V (unit diagonal, zeros above)
  double* Wz = smq + (int64_t)ldp * kNb;     // 16 x CB (W, then Z in place) / 4 x 256 partial G
  RT_INIT;
  // rows of Vs that no thread owns (>= kNT kRPT) stay zero
  for (int i = kNT * kRPT + tid; i < ldp; i += kNT)
#pragma unroll
    for (int q = 0; q < kNb; q++) Vs[i + q * ldp] = 0.0;
  for (int k0 = 0; k0 < n; k0 += kNb) {
    const int kb = min(kNb, n - k0);
    const int rows = m - k0;
    double* Ap = A + k0 + (int64_t)k0 * lda;
    // ---- 1. panel -> registers (local row li = tid + kNT u)
    double a[kRPT][kNb];
#pragma unroll
    for (int u = 0; u < kRPT; u++) {
      const int li = tid + kNT * u;
#pragma unroll
      for (int q = 0; q < kNb; q++) a[u][q] = (li < rows && q < kb) ? Ap[li + (int64_t)q * lda] : 0.0;
    }
    // ---- 2. Householder steps, one barrier per column
#pragma unroll
    for (int j = 0; j < kNb; j++) {
      {   // straight-line code for all 16 steps: the columns >= kb of a short last
          // panel are zero (tau = 0, no effect), and a column without entries
          // below the diagonal gets sc = 0 -- no (uniform) branches, whose
          // convergence barriers were 24 % of the sampled stalls (ncu r2z)
        // slot q (>= j): x . y_q over the rows below the diagonal (x = column j)
        double part[kNb];
#pragma unroll
        for (int q = 0; q < kNb; q++) part[q] = 0.0;
#pragma unroll
        for (int u = 0; u < kRPT; u++) {
          const bool below = u > 0 || tid > j;
          const double xi = below ? a[u][j] : 0.0;
#pragma unroll
          for (int q = j; q < kNb; q++) part[q] = fma(xi, a[u][q], part[q]);
        }
        double* rb = red + (j & 1) * (NW * kNb);
        double* pv = piv + (j & 1) * kNb;
        {
          // warp reduce-scatter of the 16 slots: lane L ends with slot L >> 1
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
          if ((lane & 1) == 0) rb[warp * kNb + slot] = h1;
        }
        if (tid == j) {
#pragma unroll
          for (int q = j; q < kNb; q++) pv[q] = a[0][q];
        }
        __syncthreads();
        // lane q totals slot q over the warps
        double tq = 0.0;
        if (lane < kNb) {
#pragma unroll
          for (int w = 0; w < NW; w++) tq += rb[w * kNb + lane];
        }
        const double xn2 = __shfl_sync(0xffffffffu, tq, j);
        const double alpha = pv[j];
        double t = 0.0, sc = 0.0, beta = alpha;
        if (xn2 > 0.0) {
          beta = -copysign(sqrt(alpha * alpha + xn2), alpha);
          t = (beta - alpha) / beta;
          sc = 1.0 / (alpha - beta);
        }
        // d_q = tau (y_q[j] + v . y_q), v = sc x below the pivot
        double dq = 0.0;
        if (lane > j && lane < kNb) dq = (pv[lane] + sc * tq) * t;
        double d[kNb];
#pragma unroll
        for (int q = j + 1; q < kNb; q++) d[q] = __shfl_sync(0xffffffffu, dq, q);
        if (tid == 0) {
          stau[j] = t;
          if (j < kb) J.tau[k0 + j] = t;
        }
        // t = 0 (nothing below the diagonal): sc = 0, d = 0 -- the updates are no-ops
#pragma unroll
        for (int u = 0; u < kRPT; u++) {
          const bool below = u > 0 || tid > j;
          const double vi = below ? a[u][j] * sc : 0.0;
          if (below) a[u][j] = vi;
#pragma unroll
          for (int q = j + 1; q < kNb; q++) a[u][q] = fma(-d[q], vi, a[u][q]);
        }
        if (tid == j) {
          a[0][j] = beta;
#pragma unroll
          for (int q = j + 1; q < kNb; q++) a[0][q] -= d[q];
        }
      }
    }
    // ---- 3. panel (R + reflectors) back to global memory; explicit V to shared memory
#pragma unroll
    for (int u = 0; u < kRPT; u++) {
      const int li = tid + kNT * u;
#pragma unroll
      for (int q = 0; q < kNb; q++) {
        if (li < rows && q < kb) Ap[li + (int64_t)q * lda] = a[u][q];
        if (li < ldp) Vs[li + q * ldp] = (li < rows && q < kb) ? (li > q ? a[u][q] : (li == q ? 1.0 : 0.0)) : 0.0;
      }
    }
    __syncthreads();
    RT_MARK(rt_panel);
    const int ncol = n - k0 - kb;
    if (ncol <= 0 && J.T == nullptr) continue;
    // ---- 4. T (dlarft, forward columnwise): G = V^T V on the tensor pipe (the
    // first four warps split the rows), T(i,i) = tau_i,
    // T(0:i, i) = -tau_i T(0:i,0:i) G(0:i, i)
    if (warp < 4) {
      double g00[2] = {0.0, 0.0}, g01[2] = {0.0, 0.0}, g11[2] = {0.0, 0.0};
      const double* v0 = Vs + lk + lr * ldp;
      const double* v1 = v0 + 8 * ldp;
      for (int i0 = 4 * warp; i0 < rows; i0 += 16) {   // Vs is zero in [rows, ldp), ldp = 0 (mod 4)
        const double x0 = v0[i0], x1 = v1[i0];
        dmma_r(g00, x0, x0);
        dmma_r(g01, x0, x1);
        dmma_r(g11, x1, x1);
      }
      double* gp = Wz + warp * 256;   // G(a, b) at a + 16 b
#pragma unroll
      for (int h = 0; h < 2; h++) {
        gp[lr + (2 * lk + h) * 16] = g00[h];
        gp[lr + (8 + 2 * lk + h) * 16] = g01[h];
        gp[8 + lr + (8 + 2 * lk + h) * 16] = g11[h];
      }
    }
    __syncthreads();
    for (int e = tid; e < 256; e += kNT) {
      const int ga = e & 15, gb = e >> 4;
      if (ga < gb) Wz[e] = (Wz[e] + Wz[256 + e]) + (Wz[512 + e] + Wz[768 + e]);
    }
    __syncthreads();
    if (warp == 0 && lane < kNb) {   // lane r computes row r of T, kept in registers
      const int r = lane;
      double trow[kNb];
#pragma unroll
      for (int i = 0; i < kNb; i++) {
        double v = 0.0;
        if (i < kb) {   // uniform
          double s0 = 0.0, s1 = 0.0;   // sum_{q < i} T(r, q) G(q, i)  (T(r, q) = 0 for q < r)
#pragma unroll
          for (int q = 0; q < i; q++) {
            if (q & 1) s1 = fma(trow[q], Wz[q + i * kNb], s1);
            else s0 = fma(trow[q], Wz[q + i * kNb], s0);
          }
          v = r == i ? stau[i] : (r < i ? -stau[i] * (s0 + s1) : 0.0);
        }
        trow[i] = v;
        T[r + i * kNb] = v;
      }
    }
    __syncthreads();
    if (J.T)
      for (int e = tid; e < kNb * kNb; e += kNT) J.T[(int64_t)(k0 / kNb) * kNb * kNb + e] = T[e];
    RT_MARK(rt_t);
    if (ncol <= 0) continue;
    // ---- 5. trailing update, CB columns at a time
    double* At = A + k0 + (int64_t)(k0 + kb) * lda;
    for (int cb = 0; cb < ncol; cb += CB) {
      // 5a. W = V^T A_blk: warp w owns columns cb + 8 w .. + 7
      {
        const int c0 = cb + 8 * warp;
        if (c0 < ncol) {   // warp-uniform
          const bool cok = c0 + lr < ncol;
          const double* vq0 = Vs + lk + lr * ldp;
          const double* vq1 = vq0 + 8 * ldp;
          const double* ac = At + (int64_t)(cok ? c0 + lr : c0) * lda + lk;
          double d0[2] = {0.0, 0.0}, d1[2] = {0.0, 0.0}, e0[2] = {0.0, 0.0}, e1[2] = {0.0, 0.0};
          // the warp's 8 columns are prefetched into L1 one 128-row chunk ahead
          // (9 lines per column and chunk: 72 prefetches per warp)
          const double* cbase = At + (int64_t)c0 * lda;
          const int ncw = min(8, ncol - c0);
          auto prefetch_chunk = [&](int r0) {
            for (int idx = lane; idx < 72; idx += 32) {
              const int pc = idx / 9, pr = r0 + (idx % 9) * 16;
              if (pc < ncw && pr < rows) prefetch_l1(cbase + (int64_t)pc * lda + pr);
            }
          };
          prefetch_chunk(0);
          int i0 = 0;
          for (int ch = 0; ch + 8 <= rows; ch += 128) {
            prefetch_chunk(ch + 128);
            const int iend = min(ch + 128, rows);
#pragma unroll 4
            for (; i0 + 8 <= iend; i0 += 8) {
              const double b0 = cok ? ac[i0] : 0.0;
              const double b1 = cok ? ac[i0 + 4] : 0.0;
              dmma_r(d0, vq0[i0], b0);
              dmma_r(d1, vq1[i0], b0);
              dmma_r(e0, vq0[i0 + 4], b1);
              dmma_r(e1, vq1[i0 + 4], b1);
            }
          }
          for (; i0 < rows; i0 += 4) {
            const double b0 = (cok && i0 + lk < rows) ? ac[i0] : 0.0;
            dmma_r(d0, vq0[i0], b0);
            dmma_r(d1, vq1[i0], b0);
          }
          double* w = Wz + (8 * warp) * 16;   // W(q, j) at q + 16 j (j local to the block)
#pragma unroll
          for (int h = 0; h < 2; h++) {
            w[lr + (2 * lk + h) * 16] = d0[h] + e0[h];
            w[8 + lr + (2 * lk + h) * 16] = d1[h] + e1[h];
          }
        }
      }
      __syncthreads();
      // 5b. Z(q, j) = -sum_{r <= q} T(r, q) W(r, j), in place from q = 15 down
      if (tid < CB && cb + tid < ncol) {
        double* w = Wz + tid * 16;
        double wr[kNb];
#pragma unroll
        for (int r = 0; r < kNb; r++) wr[r] = w[r];
#pragma unroll
        for (int q = 0; q < kNb; q++) {
          double s = 0.0;
#pragma unroll
          for (int r = 0; r <= q; r++) s = fma(T[r + q * kNb], wr[r], s);
          w[q] = -s;
        }
      }
      __syncthreads();
      // 5c. A_blk += V Z: 8-row tiles round-robin over the warps
      {
        const int wcb = min(CB, ncol - cb);
        const int nct = (wcb + 7) >> 3;
        double bz[NW][4];
#pragma unroll
        for (int ct = 0; ct < NW; ct++)
#pragma unroll
          for (int ks = 0; ks < 4; ks++)
            bz[ct][ks] = (ct < nct && ct * 8 + lr < wcb) ? Wz[(ks * 4 + lk) + (ct * 8 + lr) * 16] : 0.0;
        const int nrt = (rows + 7) >> 3;
        // software pipeline: the C fragments of the warp's NEXT row tile are
        // loaded before the DMMAs of the current one (the loads' L2 latency was
        // exposed once per tile)
        auto load_c = [&](int rt, auto& cc) {
          const int i = rt * 8 + lr;
          const bool iok = rt < nrt && i < rows;
#pragma unroll
          for (int ct = 0; ct < NW; ct++)
#pragma unroll
            for (int h = 0; h < 2; h++) {
              const int jj = ct * 8 + 2 * lk + h;
              cc[ct][h] = (ct < nct && iok && jj < wcb) ? At[i + (int64_t)(cb + jj) * lda] : 0.0;
            }
        };
        // (128-thread variants only: with 8 warps the 2 x 16 fragment registers spill)
        constexpr bool kPipe = NW <= 4;
        double c2[NW][2], c2n[kPipe ? NW : 1][2];
        if (kPipe) load_c(warp, c2);
        for (int rt = warp; rt < nrt; rt += NW) {
          const int i = rt * 8 + lr;
          const bool iok = i < rows;
          double av[4];
#pragma unroll
          for (int ks = 0; ks < 4; ks++) av[ks] = iok ? Vs[i + (ks * 4 + lk) * ldp] : 0.0;
          if constexpr (kPipe) load_c(rt + NW, c2n);
          else load_c(rt, c2);
#pragma unroll
          for (int ct = 0; ct < NW; ct++)
            if (ct < nct) {   // warp-uniform
#pragma unroll
              for (int ks = 0; ks < 4; ks++) dmma_r(c2[ct], av[ks], bz[ct][ks]);
            }
#pragma unroll
          for (int ct = 0; ct < NW; ct++)
#pragma unroll
            for (int h = 0; h < 2; h++) {
              const int jj = ct * 8 + 2 * lk + h;
              if (ct < nct && iok && jj < wcb) At[i + (int64_t)(cb + jj) * lda] = c2[ct][h];
              if constexpr (kPipe) c2[ct][h] = c2n[ct][h];
            }
        }
      }
      __syncthreads();
    }
    RT_MARK(rt_trail);
  }
#ifdef HM_PHASE_TIMING
  if (blockIdx.x == 0 && threadIdx.x == 0)
    printf("[qr_reg] m=%d n=%d NT=%d panel %lld T %lld trailing %lld cycles\n", m, n, kNT, rt_panel, rt_t, rt_trail);
#endif
}

template <int kNT, int kRPT, int kMinBlocks>
static void launch_one(const QrJob* d_jobs, int njobs, int max_m, cudaStream_t st) {
  constexpr int NW = kNT / 32;
  const int wz = 16 * 8 * NW > 1024 ? 16 * 8 * NW : 1024;
  const size_t bytes = ((size_t)ld4mod16(max_m) * kNb + wz) * sizeof(double);
  // the attribute is set once per (function, device): the class maximum
  ensure_smem_attr((const void*)k_qr_reg<kNT, kRPT, kMinBlocks>,
                   (int)(((size_t)ld4mod16(kNT * kRPT) * kNb + wz) * sizeof(double)));
  k_qr_reg<kNT, kRPT, kMinBlocks><<<njobs, kNT, bytes, st>>>(d_jobs);
}

// every job: n < m <= 768 (max_m = the largest m of the batch)
void launch_qr_reg(const QrJob* d_jobs, int njobs, int max_m, cudaStream_t st) {
  if (njobs <= 0) return;
  count_launch();
  if (max_m <= 128) launch_one<128, 1, 4>(d_jobs, njobs, max_m, st);
  else if (max_m <= 256) launch_one<128, 2, 3>(d_jobs, njobs, max_m, st);
  else if (max_m <= 384) launch_one<128, 3, 2>(d_jobs, njobs, max_m, st);
  // <= 512 rows: two CTAs per SM (128 registers, ~250 B of spills) for batches
  // (592 factors of 500 x 96: 2.31 -> 1.91 ms), all registers for a few factors
  // (4 factors: 0.28 vs 0.39 ms)
  else if (max_m <= 512 && njobs >= 148) launch_one<256, 2, 2>(d_jobs, njobs, max_m, st);
  else if (max_m <= 512) launch_one<256, 2, 1>(d_jobs, njobs, max_m, st);
  else launch_one<256, 3, 1>(d_jobs, njobs, max_m, st);
}

}  // namespace hm

namespace hm {

// ---------------------------------------------------------------------------
// X <- Q X, Q = H_0 ... H_{r-1} from a blocked QR with compact-WY T factors
// (Q_p = I - V_p T_p V_p^T, last panel first), ALL columns of X per pass over
// a panel: W = V_p^T X, Z = -T_p W, X += V_p Z on the FP64 tensor pipe, the
// panel staged once in shared memory (k_applyq re-reads the whole V per
// column of X: measured L2-bandwidth bound, 4.2 ms for 1184 factors of
// 760 x 128 with 40 columns).  One CTA per (job, 64 columns of X); m <= 1536.
__global__ void __launch_bounds__(256, 2) k_applyq_dmma(const ApplyQJob* __restrict__ jobs) {
  constexpr int NT = 256, NW = 8, CB = 64;
  extern __shared__ double smq[];
  __shared__ double Ts[kNb * kNb];
  const ApplyQJob J = jobs[blockIdx.x];
  const int c = J.cdyn ? *J.cdyn : J.c;
  const int cb = blockIdx.y * CB;
  if (cb >= c) return;
  const int wcb = min(CB, c - cb);
  const int m = J.m, ldv = J.ldv, ldx = J.ldx;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int lr = lane >> 2, lk = lane & 3;
  const int ldp = ld4mod16(m);
  double* Vs = smq;
  double* Wz = smq + (int64_t)ldp * kNb;
  for (int p = (J.r + kNb - 1) / kNb - 1; p >= 0; p--) {
    const int j0 = p * kNb, kb = min(kNb, J.r - j0);
    const int rows = m - j0;
    // stage the panel: explicit V (unit diagonal, zeros above / beyond rows, kb)
    {
      const double* Vp = J.V + j0 + (int64_t)j0 * ldv;
      // (read-only loads: all 16 of a row are in flight before the first store)
      for (int li = tid; li < ldp; li += NT) {
        double v[kNb];
#pragma unroll
        for (int q = 0; q < kNb; q++)
          v[q] = (li < rows && q < kb && li > q) ? __ldg(Vp + li + (int64_t)q * ldv)
                                                 : ((li == q && q < kb && li < rows) ? 1.0 : 0.0);
#pragma unroll
        for (int q = 0; q < kNb; q++) Vs[li + q * ldp] = v[q];
      }
      const double* Tp = J.T + 256 * p;
      const int q = tid & 15, r = tid >> 4;   // T(q, r), upper triangular within kb
      Ts[tid] = (q <= r && r < kb) ? __ldg(Tp + tid) : 0.0;
    }
    __syncthreads();
    double* Xt = J.X + j0 + (int64_t)cb * ldx;   // rows j0.., columns cb..
    // a. W = V^T X_blk: warp w owns columns 8 w .. 8 w + 7 of the block
    {
      const int c0 = 8 * warp;
      if (c0 < wcb) {   // warp-uniform
        const bool cok = c0 + lr < wcb;
        const double* vq0 = Vs + lk + lr * ldp;
        const double* vq1 = vq0 + 8 * ldp;
        const double* xc = Xt + (int64_t)(cok ? c0 + lr : c0) * ldx + lk;
        double d0[2] = {0.0, 0.0}, d1[2] = {0.0, 0.0}, e0[2] = {0.0, 0.0}, e1[2] = {0.0, 0.0};
        int i0 = 0;
#pragma unroll 4
        for (; i0 + 8 <= rows; i0 += 8) {
          const double b0 = cok ? xc[i0] : 0.0;
          const double b1 = cok ? xc[i0 + 4] : 0.0;
          dmma_r(d0, vq0[i0], b0);
          dmma_r(d1, vq1[i0], b0);
          dmma_r(e0, vq0[i0 + 4], b1);
          dmma_r(e1, vq1[i0 + 4], b1);
        }
        for (; i0 < rows; i0 += 4) {
          const double b0 = (cok && i0 + lk < rows) ? xc[i0] : 0.0;
          dmma_r(d0, vq0[i0], b0);
          dmma_r(d1, vq1[i0], b0);
        }
        double* w = Wz + c0 * 16;
#pragma unroll
        for (int h = 0; h < 2; h++) {
          w[lr + (2 * lk + h) * 16] = d0[h] + e0[h];
          w[8 + lr + (2 * lk + h) * 16] = d1[h] + e1[h];
        }
      }
    }
    __syncthreads();
    // b. Z(q, j) = -sum_{r >= q} T(q, r) W(r, j), in place
    if (tid < wcb) {
      double* w = Wz + tid * 16;
      double wr[kNb];
#pragma unroll
      for (int r = 0; r < kNb; r++) wr[r] = w[r];
#pragma unroll
      for (int q = 0; q < kNb; q++) {
        double s = 0.0;
#pragma unroll
        for (int r = q; r < kNb; r++) s = fma(Ts[q + r * kNb], wr[r], s);
        w[q] = -s;
      }
    }
    __syncthreads();
    // c. X_blk += V Z: 8-row tiles round-robin over the warps
    {
      const int nct = (wcb + 7) >> 3;
      double bz[NW][4];
#pragma unroll
      for (int ct = 0; ct < NW; ct++)
#pragma unroll
        for (int ks = 0; ks < 4; ks++)
          bz[ct][ks] = (ct < nct && ct * 8 + lr < wcb) ? Wz[(ks * 4 + lk) + (ct * 8 + lr) * 16] : 0.0;
      const int nrt = (rows + 7) >> 3;
      for (int rt = warp; rt < nrt; rt += NW) {
        const int i = rt * 8 + lr;
        const bool iok = i < rows;
        double av[4];
#pragma unroll
        for (int ks = 0; ks < 4; ks++) av[ks] = iok ? Vs[i + (ks * 4 + lk) * ldp] : 0.0;
        double c2[NW][2];
#pragma unroll
        for (int ct = 0; ct < NW; ct++)
#pragma unroll
          for (int h = 0; h < 2; h++) {
            const int jj = ct * 8 + 2 * lk + h;
            c2[ct][h] = (ct < nct && iok && jj < wcb) ? Xt[i + (int64_t)jj * ldx] : 0.0;
          }
#pragma unroll
        for (int ct = 0; ct < NW; ct++)
          if (ct < nct) {   // warp-uniform
#pragma unroll
            for (int ks = 0; ks < 4; ks++) dmma_r(c2[ct], av[ks], bz[ct][ks]);
          }
#pragma unroll
        for (int ct = 0; ct < NW; ct++)
#pragma unroll
          for (int h = 0; h < 2; h++) {
            const int jj = ct * 8 + 2 * lk + h;
            if (ct < nct && iok && jj < wcb) Xt[i + (int64_t)jj * ldx] = c2[ct][h];
          }
      }
    }
    __syncthreads();
  }
}

// every job: T != nullptr and m <= 1536 (max_m = the largest m); cmax = host bound of the columns
void launch_applyq_dmma(const ApplyQJob* d_jobs, int njobs, int cmax, int max_m, cudaStream_t st) {
  if (njobs <= 0 || cmax <= 0) return;
  count_launch();
  ensure_smem_attr((const void*)k_applyq_dmma, (int)(((size_t)ld4mod16(1536) * kNb + 16 * 64) * sizeof(double)));
  const size_t bytes = ((size_t)ld4mod16(max_m) * kNb + 16 * 64) * sizeof(double);
  k_applyq_dmma<<<dim3(njobs, (cmax + 63) / 64), 256, bytes, st>>>(d_jobs);
}

}  // namespace hm
