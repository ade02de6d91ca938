// Batched small SVD with the eps rank rule for TRUNC (§3 "Truncation",
// P:L336-384; rank rule = DESIGN.md §3 R1), one CTA per matrix M (p x q).
//
// Algorithm, on C = M (p >= q) or C = M^T (p < q), L x c:
//   1. Householder QR with column pivoting C P = Q R (Businger-Golub), stopped
//      at step r~ once the trailing Frobenius norm is <= delta =
//      4 u sqrt(c) ||M||_F: the dropped block only perturbs M by rounding-level
//      amounts (the backward error of the QR/GEMM that formed M).  QRCP is
//      also the classic preconditioner of one-sided Jacobi (Drmac-Veselic):
//      kernel blocks need ~6 sweeps on R^T instead of ~25 on M.
//   2. One-sided Jacobi (Hestenes) on X = R^T (c x r~), round-robin parallel
//      ordering, one warp per column pair, rotations accumulated in V (r~ x r~).
//   3. sigma_i = ||X V e_i||, descending order, smallest k with
//      sum_{i>k} sigma_i^2 <= eps^2 sum_i sigma_i^2 (tails from the bottom).
//   4. Factors: C = Q V Sigma (W/sigma)^T P^T with W = X V, so
//        p >= q: U_k = Q [V_k; 0],        V_k S_k = P W_k
//        p <  q: U_k = P W_k / sigma_k,   V_k S_k = Q [V_k S_k; 0]
//      (Q applied from the stored reflectors).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "kernels.h"

namespace hm {

static constexpr double kUs = 1.1102230246251565e-16;  // 2^-53
// fused TRUNC: no stack QR when m, n <= this (0 = always QR the thin side;
// measured: skipping it does not shorten the H-LR critical path)
static constexpr int kNoQrRows = 0;

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

// block argmax (value, lowest index on ties) and sum; results broadcast.
__device__ void bargmax_sum(double v, int idx, double s, double* redv, int* redi, double* reds,
                            double& vmax, int& imax, double& ssum) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, v, o);
    const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
    if (ov > v || (ov == v && oi < idx)) { v = ov; idx = oi; }
    s += __shfl_xor_sync(0xffffffffu, s, o);
  }
  __syncthreads();
  if (lane == 0) { redv[warp] = v; redi[warp] = idx; reds[warp] = s; }
  __syncthreads();
  if (threadIdx.x < 32) {
    v = (lane < nw) ? redv[lane] : -1.0;
    idx = (lane < nw) ? redi[lane] : 0x7fffffff;
    s = (lane < nw) ? reds[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, v, o);
      const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
      if (ov > v || (ov == v && oi < idx)) { v = ov; idx = oi; }
      s += __shfl_xor_sync(0xffffffffu, s, o);
    }
    if (lane == 0) { redv[0] = v; redi[0] = idx; reds[0] = s; }
  }
  __syncthreads();
  vmax = redv[0];
  imax = redi[0];
  ssum = reds[0];
  __syncthreads();
}

__device__ __forceinline__ int rr_pos(int k, int r, int cp) {
  return k == 0 ? 0 : ((k - 1 + r) % (cp - 1)) + 1;
}

int svd_smem_need(int p, int q) {
  const int64_t L = p > q ? p : q, c = p < q ? p : q;
  return (int)(L * c + 2 * c * c + 6 * c);
}

// SVD + rank rule + factor output of the matrix already loaded in C (L x c,
// the tall orientation of M; tr: C = M^T).  Workspace: X (c x c), V (c x c),
// tau, nrm, sig (c each), perm, order (c ints each).  Outputs per J.
__device__ void svd_core(const SvdJob& J, double eps, bool tr, int L, int c, double* C, double* X,
                         double* V, double* tau, double* nrm, double* sig, int* perm, int* order) {
  __shared__ double red[32], redv[32], reds[32];
  __shared__ int redi[32];
  __shared__ int s_rank;
  __shared__ double s_tau, s_scale;
  const int p = tr ? c : L, q = tr ? L : c;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int NT = blockDim.x, NW = NT >> 5;
  // nrm[col]: squared norm of the trailing part (rows >= j) of column col;
  // nrm2[col]: the same without row j (rows > j), both maintained exactly by
  // the update pass, so the Householder step needs no extra reduction.
  double* nrm2 = sig + 2 * (int64_t)c;
  for (int j = tid; j < c; j += NT) perm[j] = j;
  __syncthreads();
  for (int j = warp; j < c; j += NW) {
    const double* x = C + (int64_t)j * L;
    double s = 0.0, s2 = 0.0;
    for (int i = lane; i < L; i += 32) {
      s = fma(x[i], x[i], s);
      if (i > 0) s2 = fma(x[i], x[i], s2);
    }
    s = wsum(s);
    s2 = wsum(s2);
    if (lane == 0) { nrm[j] = s; nrm2[j] = s2; }
  }
  __syncthreads();
  double part = 0.0;
  for (int j = tid; j < c; j += NT) part += nrm[j];
  const double fro2 = bsum(part, red);
  const double delta2 = (16.0 * kUs * kUs) * (double)c * fro2;
  // ---------------------------------------------------------------- 1. QRCP
  int rt = 0;
  for (int j = 0; j < c && j < L; j++) {
    double v = -1.0, s = 0.0;
    int idx = 0x7fffffff;
    for (int col = j + tid; col < c; col += NT) {
      const double w = nrm[col];
      s += w;
      if (w > v) { v = w; idx = col; }
    }
    double vmax, rem;
    int piv;
    bargmax_sum(v, idx, s, redv, redi, reds, vmax, piv, rem);
    if (!(rem > delta2)) break;
    if (piv != j) {
      double* a = C + (int64_t)j * L;
      double* b = C + (int64_t)piv * L;
      for (int i = tid; i < L; i += NT) { const double t = a[i]; a[i] = b[i]; b[i] = t; }
      if (tid == 0) {
        const double t = nrm[j]; nrm[j] = nrm[piv]; nrm[piv] = t;
        const double t2 = nrm2[j]; nrm2[j] = nrm2[piv]; nrm2[piv] = t2;
        const int pt = perm[j]; perm[j] = perm[piv]; perm[piv] = pt;
      }
      __syncthreads();
    }
    double* x = C + (int64_t)j * L;
    if (tid == 0) {
      const double alpha = x[j];
      const double xn2 = nrm2[j];   // ||x[j+1:]||^2, summed directly (no cancellation)
      double t = 0.0, sc = 0.0, beta = alpha;
      if (xn2 > 0.0) {
        beta = -copysign(sqrt(alpha * alpha + xn2), alpha);
        t = (beta - alpha) / beta;
        sc = 1.0 / (alpha - beta);
      }
      x[j] = beta;
      tau[j] = t;
      s_tau = t;
      s_scale = sc;
    }
    __syncthreads();
    const double t = s_tau, sc = s_scale;
    if (t != 0.0)
      for (int i = j + 1 + tid; i < L; i += NT) x[i] *= sc;
    __syncthreads();
    for (int col = j + 1 + warp; col < c; col += NW) {
      double* y = C + (int64_t)col * L;
      double d = 0.0;
      if (t != 0.0) {
        for (int i = j + 1 + lane; i < L; i += 32) d = fma(x[i], y[i], d);
        d = (wsum(d) + y[j]) * t;
        if (lane == 0) y[j] -= d;
      }
      double nn = 0.0, nn2 = 0.0;
      for (int i = j + 1 + lane; i < L; i += 32) {
        const double yi = y[i] - d * x[i];
        y[i] = yi;
        nn = fma(yi, yi, nn);
        if (i > j + 1) nn2 = fma(yi, yi, nn2);
      }
      nn = wsum(nn);
      nn2 = wsum(nn2);
      if (lane == 0) { nrm[col] = nn; nrm2[col] = nn2; }
    }
    __syncthreads();
    rt = j + 1;
  }
  // X = R^T (c x rt), V = I
  for (int64_t e = tid; e < (int64_t)c * rt; e += NT) {
    const int col = (int)(e % c), i = (int)(e / c);
    X[e] = (col >= i) ? C[i + (int64_t)col * L] : 0.0;
  }
  for (int64_t e = tid; e < (int64_t)rt * rt; e += NT) V[e] = ((e % rt) == (e / rt)) ? 1.0 : 0.0;
  __syncthreads();
  // ---------------------------------------------------------------- 2. Jacobi
  const double tol = kUs * sqrt((double)c);
  const int cp = rt + (rt & 1);
  int sweep = 0;
  for (; sweep < 60 && rt > 1; sweep++) {
    int rot = 0;
    // one group of G lanes per column pair (G = 8/16/32 by column length):
    // shorter shuffle reductions and several pairs per warp in flight
    const int G = c <= 64 ? 8 : (c <= 128 ? 16 : 32);
    const int gl = lane & (G - 1), gpw = 32 / G;
    for (int r = 0; r < cp - 1; r++) {
      for (int base = warp * gpw; base < (cp >> 1); base += NW * gpw) {
        const int pr = base + lane / G;
        int a = 0, b = 0;
        bool act = pr < (cp >> 1);
        if (act) {
          a = rr_pos(pr, r, cp);
          b = rr_pos(cp - 1 - pr, r, cp);
          act = a < rt && b < rt;
        }
        double* x = X + (int64_t)a * c;
        double* y = X + (int64_t)b * c;
        double al = 0.0, be = 0.0, ga = 0.0;
        if (act)
          for (int i = gl; i < c; i += G) {
            const double xv = x[i], yv = y[i];
            al = fma(xv, xv, al);
            be = fma(yv, yv, be);
            ga = fma(xv, yv, ga);
          }
        for (int o = G >> 1; o > 0; o >>= 1) {   // all 32 lanes shuffle (uniform control flow)
          al += __shfl_xor_sync(0xffffffffu, al, o);
          be += __shfl_xor_sync(0xffffffffu, be, o);
          ga += __shfl_xor_sync(0xffffffffu, ga, o);
        }
        if (act && fabs(ga) > tol * sqrt(al) * sqrt(be) && fmin(al, be) > delta2) {
          const double zeta = (be - al) / (2.0 * ga);
          const double tt = copysign(1.0, zeta) / (fabs(zeta) + hypot(1.0, zeta));
          const double cs = 1.0 / sqrt(1.0 + tt * tt), sn = cs * tt;
          for (int i = gl; i < c; i += G) {
            const double xv = x[i], yv = y[i];
            x[i] = cs * xv - sn * yv;
            y[i] = sn * xv + cs * yv;
          }
          double* u = V + (int64_t)a * rt;
          double* w = V + (int64_t)b * rt;
          for (int i = gl; i < rt; i += G) {
            const double uv = u[i], wv = w[i];
            u[i] = cs * uv - sn * wv;
            w[i] = sn * uv + cs * wv;
          }
          rot = 1;
        }
      }
      __syncthreads();
    }
    if (!__syncthreads_or(rot)) break;
  }
  if (tid == 0 && J.nsweep) *J.nsweep = sweep + 1000 * rt;
  // ---------------------------------------------------------------- 3. rank
  for (int j = warp; j < rt; j += NW) {
    const double* x = X + (int64_t)j * c;
    double s = 0.0;
    for (int i = lane; i < c; i += 32) s = fma(x[i], x[i], s);
    s = wsum(s);
    if (lane == 0) sig[j] = sqrt(s);
  }
  __syncthreads();
  for (int j = tid; j < rt; j += NT) {
    const double sj = sig[j];
    int pos = 0;
    for (int i = 0; i < rt; i++) {
      const double si = sig[i];
      pos += (si > sj) || (si == sj && i < j);
    }
    order[pos] = j;
  }
  __syncthreads();
  if (tid == 0) {
    double acc = 0.0;
    for (int i = rt - 1; i >= 0; i--) { const double s = sig[order[i]]; acc += s * s; }
    int k = 0;
    if (acc > 0.0) {
      const double thr = (eps * eps) * acc;
      double tail = 0.0;
      k = rt;
      for (int kk = rt; kk >= 0; kk--) {
        if (kk < rt) { const double s = sig[order[kk]]; tail += s * s; }
        if (tail <= thr) k = kk; else break;
      }
    }
    s_rank = k;
    *J.rank = k;
  }
  __syncthreads();
  const int k = s_rank;
  if (J.sigma)
    for (int i = tid; i < c; i += NT) J.sigma[i] = (i < rt) ? sig[order[i]] : 0.0;
  // ---------------------------------------------------------------- 4. factors
  // permuted side:  out[perm[r], i] = W[r, order[i]] * f   (r < c), zero rows c..
  // Q side:         out[:, i] = Q [V[:, order[i]] * g ; 0]   (L rows), zero rows L..
  double* Pout = tr ? J.Aout : J.Bout;
  const int Pld = tr ? J.lda : J.ldb, Prows = tr ? J.ma : J.nb;
  double* Qout = tr ? J.Bout : J.Aout;
  const int Qld = tr ? J.ldb : J.lda, Qrows = tr ? J.nb : J.ma;
  for (int64_t e = tid; e < (int64_t)Prows * k; e += NT) {
    const int r = (int)(e % Prows), i = (int)(e / Prows);
    if (r >= c) Pout[r + (int64_t)i * Pld] = 0.0;
  }
  for (int64_t e = tid; e < (int64_t)c * k; e += NT) {
    const int r = (int)(e % c), i = (int)(e / c);
    const int j = order[i];
    const double f = (tr != (J.flip != 0)) ? 1.0 / sig[j] : 1.0;
    Pout[perm[r] + (int64_t)i * Pld] = X[r + (int64_t)j * c] * f;
  }
  for (int i = warp; i < k; i += NW) {
    const int j = order[i];
    const double g = (tr != (J.flip != 0)) ? sig[j] : 1.0;
    double* y = Qout + (int64_t)i * Qld;
    for (int r = lane; r < Qrows; r += 32) y[r] = (r < rt) ? V[r + (int64_t)j * rt] * g : 0.0;
    __syncwarp();
    for (int jj = rt - 1; jj >= 0; jj--) {
      const double t = tau[jj];
      if (t == 0.0) continue;
      const double* v = C + (int64_t)jj * L;
      double d = 0.0;
      for (int r = jj + 1 + lane; r < L; r += 32) d = fma(v[r], y[r], d);
      d = (wsum(d) + y[jj]) * t;
      if (lane == 0) y[jj] -= d;
      for (int r = jj + 1 + lane; r < L; r += 32) y[r] -= d * v[r];
      __syncwarp();
    }
  }
}

__global__ void k_svd(const SvdJob* __restrict__ jobs, double eps, int cap) {
  extern __shared__ double sm[];
  const SvdJob J = jobs[blockIdx.x];
  const int p = J.p, q = J.q;
  const bool tr = p < q;
  const int L = tr ? q : p, c = tr ? p : q;
  const int tid = threadIdx.x, NT = blockDim.x;
  if (c == 0) {
    if (tid == 0) *J.rank = 0;
    if (J.nsweep && tid == 0) *J.nsweep = 0;
    return;
  }
  const int64_t need = (int64_t)L * c + 2 * (int64_t)c * c + 6 * (int64_t)c;
  double* C = (need <= cap) ? sm : J.work;      // L x c, QRCP in place
  double* X = C + (int64_t)L * c;               // c x rt   (R^T, then W = X V)
  double* V = X + (int64_t)c * c;               // rt x rt  (rotations)
  double* tau = V + (int64_t)c * c;             // c
  double* nrm = tau + c;                        // c
  double* sig = nrm + c;                        // c
  int* perm = reinterpret_cast<int*>(sig + c);  // c
  int* order = perm + c;                        // c
  for (int64_t e = tid; e < (int64_t)L * c; e += NT) {
    const int i = (int)(e % L), j = (int)(e / L);
    const int mi = tr ? j : i, mj = tr ? i : j;   // entry (mi, mj) of M
    C[e] = (J.maskM && mi > mj) ? 0.0 : J.M[mi + (int64_t)mj * J.ldm];
  }
  svd_core(J, eps, tr, L, c, C, X, V, tau, nrm, sig, perm, order);
}

// In-place Householder QR (dgeqr2) of a rows x cols panel in shared memory.
__device__ void house_qr_smem(double* A, int rows, int cols, double* tau) {
  __shared__ double red[32];
  __shared__ double s_tau, s_scale;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, NT = blockDim.x, NW = NT >> 5;
  for (int j = 0; j < cols && j < rows; j++) {
    double* x = A + (int64_t)j * rows;
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
      tau[j] = t;
      s_tau = t;
      s_scale = sc;
    }
    __syncthreads();
    const double t = s_tau, sc = s_scale;
    if (t != 0.0) {
      for (int i = j + 1 + tid; i < rows; i += NT) x[i] *= sc;
      __syncthreads();
      for (int c2 = j + 1 + warp; c2 < cols; c2 += NW) {
        double* y = A + (int64_t)c2 * rows;
        double d = 0.0;
        for (int i = j + 1 + lane; i < rows; i += 32) d = fma(x[i], y[i], d);
        d = (wsum(d) + y[j]) * t;
        if (lane == 0) y[j] -= d;
        for (int i = j + 1 + lane; i < rows; i += 32) y[i] -= d * x[i];
      }
    }
    __syncthreads();
  }
}

// X (rows x k, ld ldx, global) <- H_0 ... H_{r-1} X, reflectors in shared memory.
__device__ void apply_q_smem(const double* Vr, const double* tau, int rows, int r, double* X, int ldx, int k) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, NW = blockDim.x >> 5;
  for (int col = warp; col < k; col += NW) {
    double* x = X + (int64_t)col * ldx;
    for (int j = r - 1; j >= 0; j--) {
      const double t = tau[j];
      if (t == 0.0) continue;
      const double* v = Vr + (int64_t)j * rows;
      double d = 0.0;
      for (int i = j + 1 + lane; i < rows; i += 32) d = fma(v[i], x[i], d);
      d = (wsum(d) + x[j]) * t;
      if (lane == 0) x[j] -= d;
      for (int i = j + 1 + lane; i < rows; i += 32) x[i] -= d * v[i];
      __syncwarp();
    }
  }
}

int trunc_small_need(int m, int n, int l) {
  int qa = 0, qb = 0;
  if (n >= m) qb = l < n; else qa = l < m;
  if (m <= kNoQrRows && n <= kNoQrRows) qa = qb = 0;
  const int p = qa ? l : m, q = qb ? l : n;
  const int64_t L = p > q ? p : q, c = p < q ? p : q;
  const int64_t need = (int64_t)(m + n) * l + 2 * (int64_t)l + L * c + 2 * c * c + 6 * c;
  return need > (1 << 30) ? (1 << 30) : (int)need;
}

// Fused TRUNC_eps of one small stack per CTA, everything in shared memory:
// one-sided Householder QR, M = op(A) op(B)^T in its tall orientation, the
// QRCP + Jacobi SVD of svd_core, then Q of the stack applied to the output.
__global__ void k_trunc_small(const TruncSmallJob* __restrict__ jobs, double eps) {
  extern __shared__ double sm[];
  const TruncSmallJob J = jobs[blockIdx.x];
  const int m = J.m, n = J.n, l = J.l, tid = threadIdx.x, NT = blockDim.x;
  int qa = 0, qb = 0;
  if (n >= m) qb = l < n; else qa = l < m;
  // small factors: no QR of the stack -- the column-pivoted QR of M = A B^T
  // stops at the numerical rank anyway, and the stack QR only adds
  // sequential Householder steps (latency) for these sizes
  if (m <= kNoQrRows && n <= kNoQrRows) qa = qb = 0;
  const int p = qa ? l : m, q = qb ? l : n;
  const bool tall = p >= q;
  const int L = tall ? p : q, c = tall ? q : p;
  if (c == 0 || l == 0) {
    if (tid == 0) *J.rank = 0;
    return;
  }
  double* sA = sm;
  double* sB = sA + (int64_t)m * l;
  double* tA = sB + (int64_t)n * l;
  double* tB = tA + l;
  double* C = tB + l;
  double* X = C + (int64_t)L * c;
  double* V = X + (int64_t)c * c;
  double* tau = V + (int64_t)c * c;
  double* nrm = tau + c;
  double* sig = nrm + c;
  int* perm = reinterpret_cast<int*>(sig + c);
  int* order = perm + c;
  for (int64_t e = tid; e < (int64_t)m * l; e += NT) sA[e] = J.A[e];
  for (int64_t e = tid; e < (int64_t)n * l; e += NT) sB[e] = J.B[e];
  __syncthreads();
  if (qa) house_qr_smem(sA, m, l, tA);
  if (qb) house_qr_smem(sB, n, l, tB);
  // Mt = op(A) op(B)^T (tall) or op(B) op(A)^T
  for (int64_t e = tid; e < (int64_t)L * c; e += NT) {
    const int i = (int)(e % L), j = (int)(e / L);
    const int ia = tall ? i : j, ib = tall ? j : i;   // row of op(A), row of op(B)
    double s = 0.0;
    for (int k = 0; k < l; k++) {
      const double a = (qa && ia > k) ? 0.0 : sA[ia + (int64_t)k * m];
      const double b = (qb && ib > k) ? 0.0 : sB[ib + (int64_t)k * n];
      s = fma(a, b, s);
    }
    C[e] = s;
  }
  __syncthreads();
  SvdJob S{};
  S.rank = J.rank;
  S.sigma = J.sigma;
  S.flip = tall ? 0 : 1;
  S.Aout = tall ? J.Aout : J.Bout;
  S.lda = tall ? m : n;
  S.ma = S.lda;
  S.Bout = tall ? J.Bout : J.Aout;
  S.ldb = tall ? n : m;
  S.nb = S.ldb;
  svd_core(S, eps, false, L, c, C, X, V, tau, nrm, sig, perm, order);
  __syncthreads();
  const int k = *J.rank;
  if (qa) apply_q_smem(sA, tA, m, l, J.Aout, m, k);
  if (qb) apply_q_smem(sB, tB, n, l, J.Bout, n, k);
}

void launch_trunc_small(const TruncSmallJob* d_jobs, int njobs, double eps, int cap, cudaStream_t st) {
  if (njobs <= 0) return;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_trunc_small, cudaFuncAttributeMaxDynamicSharedMemorySize, 26 * 1024 * 8);
    attr = true;
  }
  count_launch();
  // small stacks: one warp per stack (barriers of a 1-warp CTA are nearly
  // free, and many stacks share an SM); larger: 128 / 256 threads
  // (measured on B200: 32 or 128 threads for the small buckets is slower --
  // the L x c loops lose more than the cheaper barriers gain)
  const int threads = 256;
  k_trunc_small<<<njobs, threads, (size_t)cap * 8, st>>>(d_jobs, eps);
}

int svd_smem_capacity() { return 26 * 1024; }

void launch_svd(const SvdJob* d_jobs, int njobs, double eps, int cap, cudaStream_t st) {
  if (njobs <= 0) return;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_svd, cudaFuncAttributeMaxDynamicSharedMemorySize, svd_smem_capacity() * 8);
    attr = true;
  }
  if (cap > svd_smem_capacity()) cap = svd_smem_capacity();
  const int threads = (cap == 0 || cap > 8 * 1024) ? 512 : 256;
  count_launch();
  k_svd<<<njobs, threads, (size_t)cap * 8, st>>>(d_jobs, eps, cap);
}

}  // namespace hm
