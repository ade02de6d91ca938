// Batched H x thin-dense products (addeval / addevaltrans, Fig. 1
// P:L300-334) for the addproduct evaluations of one level.
//
// One CTA per EvalJob (the leaves [leaf_begin, leaf_end) of one block of X or
// Y, in DFS order); the CTA owns its output panel (distinct stack columns), so
// no atomics and bit-reproducible results.  Every leaf is streamed through
// shared memory in 64-row tiles with coalesced loads, and the products run
// from shared memory into register accumulators:
//   dense leaf     out[i, j] += coef sum_p op(N)(i, p) V(p, j)
//   low-rank leaf  T = F2^T V (k x w, reduced over F2's rows in 64-row chunks),
//                  out += coef F1 T            (F1 = A, F2 = B; swapped for ^T)
//   V = I          the leaf itself (dense tile copy / F1 F2^T) added into out.
// Column blocks of 32 (w > 32) and rank chunks of 32 (k > 32) loop.
#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels.h"

namespace hm {

namespace {
constexpr int kT = 64;    // tile rows (out rows) and K chunk
constexpr int kW = 32;    // column block (of V / out) and rank chunk
constexpr int kNT = 256;
constexpr int kLdS = kT + 1;   // S: 64 x 64 tile, (i, p) at i + p * 65
constexpr int kLdV = kW + 1;   // Vt: (p, j) at p * 33 + j ; Ts: (q, j) at q * 33 + j
constexpr int kSmem = kT * kLdS + kT * kLdV + kW * kLdV;

__device__ __forceinline__ double vat(const EvalJob& J, int p, int j) {
  return J.vtrans ? J.V[j + (int64_t)p * J.ldv] : J.V[p + (int64_t)j * J.ldv];
}

// Vt[p][j] = V(vrow + p0 + p, j0 + j), zero padded to 64 x 32
__device__ __forceinline__ void stage_v(const EvalJob& J, int vrow, int p0, int pc, int j0, int wc, double* Vt) {
  const int tid = threadIdx.x;
  if (!J.vtrans) {
    for (int e = tid; e < kT * kW; e += kNT) {
      const int p = e % kT, j = e / kT;
      Vt[p * kLdV + j] = (p < pc && j < wc) ? J.V[(vrow + p0 + p) + (int64_t)(j0 + j) * J.ldv] : 0.0;
    }
  } else {
    for (int e = tid; e < kT * kW; e += kNT) {
      const int j = e % kW, p = e / kW;
      Vt[p * kLdV + j] = (p < pc && j < wc) ? J.V[(j0 + j) + (int64_t)(vrow + p0 + p) * J.ldv] : 0.0;
    }
  }
}

// out[orow + i0 + i, ocol + j0 + j] += coef * acc  (thread: i = tid & 63, j = (tid >> 6) + 4 u, u < NU)
template <int NU>
__device__ __forceinline__ void store_acc(const EvalJob& J, int orow, int ocol, int i0, int mc, int j0, int wc,
                                          const double (&acc)[NU]) {
  const int i = threadIdx.x & (kT - 1), jg = threadIdx.x >> 6;
  if (i >= mc) return;
  double* o = J.out + (orow + i0 + i);
#pragma unroll
  for (int u = 0; u < NU; u++) {
    const int j = jg + 4 * u;
    if (j < wc) {
      double* d = o + (int64_t)(ocol + j0 + j) * J.ldo;
      *d = fma(J.coef, acc[u], *d);
    }
  }
}

// acc += S(i, 0:kc) * W(0:kc, j), S at i + p * 65 (shared), W at p * 33 + j (shared)
template <int NU>
__device__ __forceinline__ void tile_mma(const double* S, const double* W, int kc, double (&acc)[NU]) {
  const int i = threadIdx.x & (kT - 1), jg = threadIdx.x >> 6;
#pragma unroll 4
  for (int p = 0; p < kc; p++) {
    const double s = S[i + p * kLdS];
    const double* w = W + p * kLdV + jg;
#pragma unroll
    for (int u = 0; u < NU; u++) acc[u] = fma(s, w[4 * u], acc[u]);
  }
}

template <int NU>
__device__ void dense_tiles(const EvalJob& J, const LeafDesc& L, int orow, int vrow, int mo, int ko, int j0, int wc,
                            double* S, double* Vt) {
  const int tid = threadIdx.x;
  const int ldn = L.m;
  for (int i0 = 0; i0 < mo; i0 += kT) {
    const int mc = min(kT, mo - i0);
    double acc[NU];
#pragma unroll
    for (int u = 0; u < NU; u++) acc[u] = 0.0;
    for (int p0 = 0; p0 < ko; p0 += kT) {
      const int pc = min(kT, ko - p0);
      // S(i, p) = op(N)(i0 + i, p0 + p)
      if (!J.trans) {
        for (int e = tid; e < kT * kT; e += kNT) {
          const int i = e % kT, p = e / kT;
          S[i + p * kLdS] = (i < mc && p < pc) ? L.A[(i0 + i) + (int64_t)(p0 + p) * ldn] : 0.0;
        }
      } else {
        for (int e = tid; e < kT * kT; e += kNT) {
          const int p = e % kT, i = e / kT;
          S[i + p * kLdS] = (i < mc && p < pc) ? L.A[(p0 + p) + (int64_t)(i0 + i) * ldn] : 0.0;
        }
      }
      stage_v(J, vrow, p0, pc, j0, wc, Vt);
      __syncthreads();
      tile_mma<NU>(S, Vt, pc, acc);
      __syncthreads();
    }
    store_acc<NU>(J, orow, 0, i0, mc, j0, wc, acc);
  }
}

__device__ void eval_dense(const EvalJob& J, const LeafDesc& L, int orow, int vrow, int mo, int ko, double* S,
                           double* Vt) {
  for (int j0 = 0; j0 < J.w; j0 += kW) {
    const int wc = min(kW, J.w - j0);
    if (wc <= 8) dense_tiles<2>(J, L, orow, vrow, mo, ko, j0, wc, S, Vt);
    else if (wc <= 16) dense_tiles<4>(J, L, orow, vrow, mo, ko, j0, wc, S, Vt);
    else dense_tiles<8>(J, L, orow, vrow, mo, ko, j0, wc, S, Vt);
  }
}

// out(orow + i, ocol + j) += coef sum_q F1(i, q) Ts(q, j) for the rank chunk in Ts
template <int NU>
__device__ void apply_f1_t(const EvalJob& J, const double* F1, int ld1, int mo, int q0, int kc, int orow, int ocol,
                           int j0, int wc, double* S, const double* Ts) {
  const int tid = threadIdx.x;
  for (int i0 = 0; i0 < mo; i0 += kT) {
    const int mc = min(kT, mo - i0);
    for (int e = tid; e < kT * kW; e += kNT) {
      const int i = e % kT, q = e / kT;
      S[i + q * kLdS] = (i < mc && q < kc) ? F1[(i0 + i) + (int64_t)(q0 + q) * ld1] : 0.0;
    }
    __syncthreads();
    double acc[NU];
#pragma unroll
    for (int u = 0; u < NU; u++) acc[u] = 0.0;
    tile_mma<NU>(S, Ts, kc, acc);
    store_acc<NU>(J, orow, ocol, i0, mc, j0, wc, acc);
    __syncthreads();
  }
}

__device__ void apply_f1(const EvalJob& J, const double* F1, int ld1, int mo, int q0, int kc, int orow, int ocol,
                         int j0, int wc, double* S, const double* Ts) {
  if (wc <= 8) apply_f1_t<2>(J, F1, ld1, mo, q0, kc, orow, ocol, j0, wc, S, Ts);
  else if (wc <= 16) apply_f1_t<4>(J, F1, ld1, mo, q0, kc, orow, ocol, j0, wc, S, Ts);
  else apply_f1_t<8>(J, F1, ld1, mo, q0, kc, orow, ocol, j0, wc, S, Ts);
}

__device__ void eval_lowrank(const EvalJob& J, const LeafDesc& L, int orow, int vrow, int mo, int ko, double* S,
                             double* Vt, double* Ts) {
  const int tid = threadIdx.x;
  const double* F1 = J.trans ? L.B : L.A;
  const int ld1 = J.trans ? L.n : L.m;
  const double* F2 = J.trans ? L.A : L.B;
  const int ld2 = J.trans ? L.m : L.n;
  for (int j0 = 0; j0 < J.w; j0 += kW) {
    const int wc = min(kW, J.w - j0);
    for (int q0 = 0; q0 < L.k; q0 += kW) {
      const int kc = min(kW, L.k - q0);
      // T(q, j) = sum_p F2(p, q0 + q) V(vrow + p, j0 + j); thread: q = tid & 31, j = warp + 8 u
      const int q = tid & 31, jw = tid >> 5;
      double t[4] = {0.0, 0.0, 0.0, 0.0};
      for (int p0 = 0; p0 < ko; p0 += kT) {
        const int pc = min(kT, ko - p0);
        for (int e = tid; e < kT * kW; e += kNT) {   // S2(q, p) at q + p * 33 (conflict-free reads)
          const int p = e % kT, qq = e / kT;
          S[qq + p * kLdV] = (p < pc && qq < kc) ? F2[(p0 + p) + (int64_t)(q0 + qq) * ld2] : 0.0;
        }
        stage_v(J, vrow, p0, pc, j0, wc, Vt);
        __syncthreads();
#pragma unroll 4
        for (int p = 0; p < pc; p++) {
          const double f = S[q + p * kLdV];
          const double* v = Vt + p * kLdV + jw;
#pragma unroll
          for (int u = 0; u < 4; u++) t[u] = fma(f, v[8 * u], t[u]);
        }
        __syncthreads();
      }
#pragma unroll
      for (int u = 0; u < 4; u++) Ts[q * kLdV + jw + 8 * u] = t[u];
      __syncthreads();
      apply_f1(J, F1, ld1, mo, q0, kc, orow, 0, j0, wc, S, Ts);
    }
  }
}

// V = I: out(orow + i, vrow + p) += coef op(L)(i, p)
__device__ void eval_identity(const EvalJob& J, const LeafDesc& L, int orow, int vrow, int mo, int ko, double* S,
                              double* Ts) {
  const int tid = threadIdx.x;
  if (L.kind == 2) {
    const int ldn = L.m;
    if (!J.trans) {
      for (int64_t e = tid; e < (int64_t)mo * ko; e += kNT) {
        const int i = (int)(e % mo), p = (int)(e / mo);
        double* d = J.out + (orow + i) + (int64_t)(vrow + p) * J.ldo;
        *d = fma(J.coef, L.A[i + (int64_t)p * ldn], *d);
      }
    } else {
      for (int i0 = 0; i0 < mo; i0 += kT)
        for (int p0 = 0; p0 < ko; p0 += kT) {
          const int mc = min(kT, mo - i0), pc = min(kT, ko - p0);
          for (int e = tid; e < kT * kT; e += kNT) {   // S(i, p) = N(p0 + p, i0 + i)
            const int p = e % kT, i = e / kT;
            if (p < pc && i < mc) S[i + p * kLdS] = L.A[(p0 + p) + (int64_t)(i0 + i) * ldn];
          }
          __syncthreads();
          for (int e = tid; e < kT * kT; e += kNT) {
            const int i = e % kT, p = e / kT;
            if (i < mc && p < pc) {
              double* d = J.out + (orow + i0 + i) + (int64_t)(vrow + p0 + p) * J.ldo;
              *d = fma(J.coef, S[i + p * kLdS], *d);
            }
          }
          __syncthreads();
        }
    }
    __syncthreads();
    return;
  }
  if (L.k <= 0) return;
  const double* F1 = J.trans ? L.B : L.A;
  const int ld1 = J.trans ? L.n : L.m;
  const double* F2 = J.trans ? L.A : L.B;
  const int ld2 = J.trans ? L.m : L.n;
  for (int j0 = 0; j0 < ko; j0 += kW) {        // output columns = rows of F2
    const int wc = min(kW, ko - j0);
    for (int q0 = 0; q0 < L.k; q0 += kW) {
      const int kc = min(kW, L.k - q0);
      for (int e = tid; e < kW * kW; e += kNT) {   // Ts(q, j) = F2(j0 + j, q0 + q)
        const int j = e % kW, q = e / kW;
        Ts[q * kLdV + j] = (j < wc && q < kc) ? F2[(j0 + j) + (int64_t)(q0 + q) * ld2] : 0.0;
      }
      __syncthreads();
      apply_f1(J, F1, ld1, mo, q0, kc, orow, vrow, j0, wc, S, Ts);
    }
  }
}
}  // namespace

__device__ void eval_range(const EvalJob& J, int lb, int le, double* sm) {
  double* S = sm;
  double* Vt = S + kT * kLdS;
  double* Ts = Vt + kT * kLdV;
  for (int li = lb; li < le; li++) {
    __syncthreads();   // the previous leaf's output writes are visible to every thread
    const LeafDesc L = J.leaves[li];
    const int ro = L.row0 - J.t0, co = L.col0 - J.s0;   // offsets inside block (t,s)
    const int orow = J.trans ? co : ro;                 // out rows
    const int vrow = J.trans ? ro : co;                 // V rows (or out columns when V = I)
    const int mo = J.trans ? L.n : L.m;                 // rows of op(L)
    const int ko = J.trans ? L.m : L.n;                 // cols of op(L)
    if (J.videntity) eval_identity(J, L, orow, vrow, mo, ko, S, Ts);
    else if (L.kind == 2) eval_dense(J, L, orow, vrow, mo, ko, S, Vt);
    else if (L.k > 0) eval_lowrank(J, L, orow, vrow, mo, ko, S, Vt, Ts);
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kNT) k_eval2(const EvalJob* __restrict__ jobs) {
  extern __shared__ double sm[];
  const EvalJob J = jobs[blockIdx.x];
  eval_range(J, J.leaf_begin, J.leaf_end, sm);
}

// ------------------------------------------------------------------ TRSM
// Triangular solve through the H-structure on one thin panel per CTA (host
// step lists, see kernels.h): (a) V[r0:r0+m, :] <- T^-1 V with T a dense
// lower-triangular leaf block (m <= 64), column-oriented substitution in
// shared memory -- one barrier per pivot row, all (row, column) updates of a
// step in parallel; (b) V -= op(H) V over a leaf range with the eval tiles.
constexpr int kTrsmCols = 96;                          // panel columns per substitution chunk
constexpr int kTrsmSmem = kT * kLdS + kT + kTrsmCols * (kT + 1);
constexpr int kTrsmShared = kTrsmSmem > kSmem ? kTrsmSmem : kSmem;

__global__ void __launch_bounds__(kNT) k_trsm2(const TrsmJob* __restrict__ jobs, const TrsmStep* __restrict__ steps,
                                               const LeafDesc* __restrict__ leaves) {
  extern __shared__ double sm[];
  const TrsmJob J = jobs[blockIdx.x];
  const int tid = threadIdx.x;
  for (int si = J.step0; si < J.step1; si++) {
    const TrsmStep S = steps[si];
    if (S.kind == 0 && S.m > kT) {
      // leaf clusters larger than 64 rows (leaf size > 64): plain substitution
      // in global memory, one thread per column
      double* v = J.V + S.r0;
      for (int col = tid; col < J.ncols; col += kNT) {
        double* x = v + (int64_t)col * J.ldv;
        for (int i = 0; i < S.m; i++) {
          double acc = x[i];
          for (int p = 0; p < i; p++)
            acc = fma(-(S.trans ? S.P[p + (int64_t)i * S.ld] : S.P[i + (int64_t)p * S.ld]), x[p], acc);
          x[i] = S.unit ? acc : acc / S.P[i + (int64_t)i * S.ld];
        }
      }
      __syncthreads();
    } else if (S.kind == 0) {
      const int m = S.m;
      double* tri = sm;                  // T(i, p) at i + p * 65
      double* dinv = tri + kT * kLdS;    // 1 / T(i, i)
      double* xs = dinv + kT;            // panel chunk (i, c) at c * (m + 1) + i
      double* v = J.V + S.r0;
      for (int e = tid; e < m * m; e += kNT) {
        const int i = e % m, j = e / m;
        tri[i + j * kLdS] = S.trans ? S.P[j + (int64_t)i * S.ld] : S.P[i + (int64_t)j * S.ld];
      }
      __syncthreads();
      for (int i = tid; i < m; i += kNT) dinv[i] = S.unit ? 1.0 : 1.0 / tri[i + i * kLdS];
      const int ldx = m + 1;
      for (int c0 = 0; c0 < J.ncols; c0 += kTrsmCols) {
        const int cc = min(kTrsmCols, J.ncols - c0);
        for (int e = tid; e < m * cc; e += kNT) {
          const int i = e % m, c = e / m;
          xs[c * ldx + i] = v[i + (int64_t)(c0 + c) * J.ldv];
        }
        __syncthreads();
        // x_p final = x_p * dinv_p; rows i > p: x_i -= T(i, p) x_p dinv_p
        for (int p = 0; p < m - 1; p++) {
          const int rows = m - 1 - p;
          const double dp = dinv[p];
          for (int e = tid; e < rows * cc; e += kNT) {
            const int i = p + 1 + e % rows, c = e / rows;
            xs[c * ldx + i] = fma(-tri[i + p * kLdS] * dp, xs[c * ldx + p], xs[c * ldx + i]);
          }
          __syncthreads();
        }
        for (int e = tid; e < m * cc; e += kNT) {
          const int i = e % m, c = e / m;
          v[i + (int64_t)(c0 + c) * J.ldv] = xs[c * ldx + i] * dinv[i];
        }
        __syncthreads();
      }
    } else {
      EvalJob E{};
      E.leaves = leaves;
      E.trans = S.trans;
      E.t0 = J.panel0;
      E.s0 = J.panel0;
      E.coef = -1.0;
      E.out = J.V;
      E.ldo = J.ldv;
      E.w = J.ncols;
      E.V = J.V;
      E.ldv = J.ldv;
      eval_range(E, S.lb, S.le, sm);
    }
  }
}

void launch_trsm2(const TrsmJob* d_jobs, int njobs, const TrsmStep* d_steps, const LeafDesc* leaves, cudaStream_t st) {
  if (njobs <= 0) return;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_trsm2, cudaFuncAttributeMaxDynamicSharedMemorySize, kTrsmShared * 8);
    attr = true;
  }
  count_launch();
  k_trsm2<<<njobs, kNT, (size_t)kTrsmShared * 8, st>>>(d_jobs, d_steps, leaves);
}

void launch_eval2(const EvalJob* d_jobs, int njobs, cudaStream_t st) {
  if (njobs <= 0) return;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_eval2, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem * 8);
    attr = true;
  }
  count_launch();
  k_eval2<<<njobs, kNT, (size_t)kSmem * 8, st>>>(d_jobs);
}

}  // namespace hm
