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
constexpr int kT = 64;     // tile rows (out rows) and K chunk
constexpr int kW = 32;     // column block (of V / out) and rank chunk
constexpr int kNT = 256;
// Shared-memory leading dimensions = 4 (mod 16): the DMMA fragment loads (8
// rows x 4 k per warp, lanes (r, k) = (lane >> 2, lane & 3)) and the staging
// stores (consecutive elements) are both bank-conflict free.
constexpr int kLd = 68;
constexpr int kLdJ = 36;
constexpr int kLdS = kT + 1;              // identity path / TRSM tiles: (i, p) at i + p * 65
constexpr int kSmemS = kT * kLd;          // S: 64 x 64 operand tile, either orientation
constexpr int kSmemV = kT * kLdJ;         // V: 64 x 32 (j + p * 36) or 32 x 64 (p + j * 68)
constexpr int kSmemT = kW * kLdJ;         // Ts: (q, j) at j + q * 36
constexpr int kSmem = kSmemS + kSmemV + kSmemT;
static_assert(kW * kLd <= kSmemV, "V tile");
static_assert(kT * kLdS <= kSmemS, "identity tile");

// Asynchronous global -> shared copy of one double (LDGSTS; zero fill when
// !ok, the source is then not read): every staging load of a tile is in
// flight at once instead of one load -> store round trip per element.
__device__ __forceinline__ void cp8(double* dst, const double* src, bool ok) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(src), "r"(ok ? 8 : 0) : "memory");
}
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// D(8x8) += A(8x4) B(4x8) in FP64 on the tensor pipe (DMMA.8x8x4).  Fragments
// (PTX m8n8k4 .f64): a = A(lane >> 2, lane & 3), b = B(lane & 3, lane >> 2),
// d = D(lane >> 2, 2 (lane & 3) + {0, 1}).
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d[0]), "+d"(d[1])
      : "d"(a), "d"(b));
}

// Warp tiling of an (8 MT) x (8 NCT) output over the 8 warps: each warp owns
// RTW x CTW 8x8 tiles (row group rg, column group cg).
template <int MT, int NCT>
struct WarpTiling {
  static constexpr int RTW = (MT == 8 && NCT == 4) ? 2 : 1;
  static constexpr int CTW = (NCT == 4 || (NCT == 2 && MT == 8)) ? 2 : 1;
  static constexpr int RG = MT / RTW;
  static constexpr int CG = NCT / CTW;
};

// acc += A(8 MT x kc) B(kc x 8 NCT), A(i, p) = As[i ars + p acs], B(p, j) =
// Bs[p brs + j bcs] (shared memory, zero padded to kc rounded up to 4).
template <int MT, int NCT>
__device__ __forceinline__ void tile_dmma(const double* As, int ars, int acs, const double* Bs, int brs, int bcs,
                                          int kc, double (&acc)[WarpTiling<MT, NCT>::RTW * WarpTiling<MT, NCT>::CTW][2]) {
  using WT = WarpTiling<MT, NCT>;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (warp >= WT::RG * WT::CG) return;
  const int rg = warp % WT::RG, cg = warp / WT::RG;
  const int lr = lane >> 2, lk = lane & 3;
  const double* a0 = As + (rg * WT::RTW * 8 + lr) * ars + lk * acs;
  const double* b0 = Bs + lk * brs + (cg * WT::CTW * 8 + lr) * bcs;
#pragma unroll 4
  for (int k0 = 0; k0 < kc; k0 += 4) {
    double a[WT::RTW], b[WT::CTW];
#pragma unroll
    for (int r = 0; r < WT::RTW; r++) a[r] = a0[r * 8 * ars + k0 * acs];
#pragma unroll
    for (int c = 0; c < WT::CTW; c++) b[c] = b0[c * 8 * bcs + k0 * brs];
#pragma unroll
    for (int r = 0; r < WT::RTW; r++)
#pragma unroll
      for (int c = 0; c < WT::CTW; c++) dmma(acc[r * WT::CTW + c], a[r], b[c]);
  }
}

template <int MT, int NCT>
__device__ __forceinline__ void acc_zero(double (&acc)[WarpTiling<MT, NCT>::RTW * WarpTiling<MT, NCT>::CTW][2]) {
#pragma unroll
  for (int t = 0; t < WarpTiling<MT, NCT>::RTW * WarpTiling<MT, NCT>::CTW; t++) acc[t][0] = acc[t][1] = 0.0;
}

// The old values of the warp's output fragments, loaded BEFORE the tile is
// computed (the read-modify-write of store_acc was k_eval2's long-scoreboard
// stall: the load latency now overlaps the staging and the DMMA work).
template <int NCT>
__device__ __forceinline__ void load_out(const EvalJob& J, int orow, int ocol, int i0, int mc, int j0, int wc,
                                         double (&old)[WarpTiling<8, NCT>::RTW * WarpTiling<8, NCT>::CTW][2]) {
  using WT = WarpTiling<8, NCT>;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int t = 0; t < WT::RTW * WT::CTW; t++) old[t][0] = old[t][1] = 0.0;
  if (warp >= WT::RG * WT::CG) return;
  const int rg = warp % WT::RG, cg = warp / WT::RG;
#pragma unroll
  for (int r = 0; r < WT::RTW; r++) {
    const int i = (rg * WT::RTW + r) * 8 + (lane >> 2);
    if (i >= mc) continue;
    const double* o = J.out + (orow + i0 + i);
#pragma unroll
    for (int c = 0; c < WT::CTW; c++)
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int j = (cg * WT::CTW + c) * 8 + 2 * (lane & 3) + h;
        if (j < wc) old[r * WT::CTW + c][h] = o[(int64_t)(ocol + j0 + j) * J.ldo];
      }
  }
}

// out[orow + i0 + i, ocol + j0 + j] = old + coef * D(i, j) for i < mc, j < wc
template <int NCT>
__device__ __forceinline__ void store_acc_old(const EvalJob& J, int orow, int ocol, int i0, int mc, int j0, int wc,
                                              const double (&acc)[WarpTiling<8, NCT>::RTW * WarpTiling<8, NCT>::CTW][2],
                                              const double (&old)[WarpTiling<8, NCT>::RTW * WarpTiling<8, NCT>::CTW][2]) {
  using WT = WarpTiling<8, NCT>;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (warp >= WT::RG * WT::CG) return;
  const int rg = warp % WT::RG, cg = warp / WT::RG;
#pragma unroll
  for (int r = 0; r < WT::RTW; r++) {
    const int i = (rg * WT::RTW + r) * 8 + (lane >> 2);
    if (i >= mc) continue;
    double* o = J.out + (orow + i0 + i);
#pragma unroll
    for (int c = 0; c < WT::CTW; c++)
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int j = (cg * WT::CTW + c) * 8 + 2 * (lane & 3) + h;
        if (j < wc) o[(int64_t)(ocol + j0 + j) * J.ldo] = fma(J.coef, acc[r * WT::CTW + c][h], old[r * WT::CTW + c][h]);
      }
  }
}

// out[orow + i0 + i, ocol + j0 + j] += coef * D(i, j) for i < mc, j < wc
template <int NCT>
__device__ __forceinline__ void store_acc(const EvalJob& J, int orow, int ocol, int i0, int mc, int j0, int wc,
                                          const double (&acc)[WarpTiling<8, NCT>::RTW * WarpTiling<8, NCT>::CTW][2]) {
  using WT = WarpTiling<8, NCT>;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (warp >= WT::RG * WT::CG) return;
  const int rg = warp % WT::RG, cg = warp / WT::RG;
#pragma unroll
  for (int r = 0; r < WT::RTW; r++) {
    const int i = (rg * WT::RTW + r) * 8 + (lane >> 2);
    if (i >= mc) continue;
    double* o = J.out + (orow + i0 + i);
#pragma unroll
    for (int c = 0; c < WT::CTW; c++)
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int j = (cg * WT::CTW + c) * 8 + 2 * (lane & 3) + h;
        if (j < wc) {
          double* d = o + (int64_t)(ocol + j0 + j) * J.ldo;
          *d = fma(J.coef, acc[r * WT::CTW + c][h], *d);
        }
      }
  }
}

// V(vrow + p0 + p, j0 + j) for p < 64, j < 32, zero padded; the B operand
// descriptor (brs, bcs) of the layout used.
__device__ __forceinline__ void stage_v(const EvalJob& J, int vrow, int p0, int pc, int j0, int wc, double* Vs,
                                        int& brs, int& bcs) {
  const int tid = threadIdx.x;
  const int pcp = (pc + 3) & ~3;   // rows [pc, pcp) zero (read by the k loop); columns >= wc and rows >= pcp
                                   // are left stale: they only reach output columns that are discarded
  if (!J.vtrans) {   // p contiguous in global: Vs[p + j * 68]
    for (int e = tid; e < kT * wc; e += kNT) {
      const int p = e & (kT - 1), j = e >> 6;
      if (p >= pcp) continue;
      const bool ok = p < pc;
      cp8(Vs + p + j * kLd, ok ? J.V + (vrow + p0 + p) + (int64_t)(j0 + j) * J.ldv : J.V, ok);
    }
    brs = 1;
    bcs = kLd;
  } else {           // j contiguous in global: Vs[j + p * 36]
    for (int e = tid; e < kW * pcp; e += kNT) {
      const int j = e & (kW - 1), p = e >> 5;
      if (j >= wc) continue;
      const bool ok = p < pc;
      cp8(Vs + j + p * kLdJ, ok ? J.V + (j0 + j) + (int64_t)(vrow + p0 + p) * J.ldv : J.V, ok);
    }
    brs = kLdJ;
    bcs = 1;
  }
}

template <int NCT>
__device__ void dense_tiles(const EvalJob& J, const LeafDesc& L, int orow, int vrow, int mo, int ko, int j0, int wc,
                            double* S, double* Vs) {
  const int tid = threadIdx.x;
  const int ldn = L.m;
  for (int i0 = 0; i0 < mo; i0 += kT) {
    const int mc = min(kT, mo - i0);
    double acc[WarpTiling<8, NCT>::RTW * WarpTiling<8, NCT>::CTW][2];
    double old[WarpTiling<8, NCT>::RTW * WarpTiling<8, NCT>::CTW][2];
    acc_zero<8, NCT>(acc);
    load_out<NCT>(J, orow, 0, i0, mc, j0, wc, old);
    for (int p0 = 0; p0 < ko; p0 += kT) {
      const int pc = min(kT, ko - p0), pcp = (pc + 3) & ~3;
      int ars, acs, brs, bcs;
      // S: rows >= mc stale (their output rows are discarded), k columns [pc, pcp) zero
      if (!J.trans) {   // op(N)(i, p) = N(i, p), i contiguous: S[i + p * 68]
        for (int e = tid; e < kT * pcp; e += kNT) {
          const int i = e & (kT - 1), p = e >> 6;
          if (i >= mc) continue;
          const bool ok = p < pc;
          cp8(S + i + p * kLd, ok ? L.A + (i0 + i) + (int64_t)(p0 + p) * ldn : L.A, ok);
        }
        ars = 1;
        acs = kLd;
      } else {          // op(N)(i, p) = N(p, i), p contiguous: S[p + i * 68]
        for (int e = tid; e < kT * mc; e += kNT) {
          const int p = e & (kT - 1), i = e >> 6;
          if (p >= pcp) continue;
          const bool ok = p < pc;
          cp8(S + p + i * kLd, ok ? L.A + (p0 + p) + (int64_t)(i0 + i) * ldn : L.A, ok);
        }
        ars = kLd;
        acs = 1;
      }
      stage_v(J, vrow, p0, pc, j0, wc, Vs, brs, bcs);
      cp_wait();
      __syncthreads();
      tile_dmma<8, NCT>(S, ars, acs, Vs, brs, bcs, (pc + 3) & ~3, acc);
      __syncthreads();
    }
    store_acc_old<NCT>(J, orow, 0, i0, mc, j0, wc, acc, old);
  }
}

__device__ void eval_dense(const EvalJob& J, const LeafDesc& L, int orow, int vrow, int mo, int ko, double* S,
                           double* Vs) {
  for (int j0 = 0; j0 < J.w; j0 += kW) {
    const int wc = min(kW, J.w - j0);
    if (wc <= 8) dense_tiles<1>(J, L, orow, vrow, mo, ko, j0, wc, S, Vs);
    else if (wc <= 16) dense_tiles<2>(J, L, orow, vrow, mo, ko, j0, wc, S, Vs);
    else dense_tiles<4>(J, L, orow, vrow, mo, ko, j0, wc, S, Vs);
  }
}

// out(orow + i, ocol + j0 + j) += coef sum_q F1(i, q0 + q) Ts(q, j), Ts(q, j) at j + q * 36
template <int NCT>
__device__ void apply_f1_t(const EvalJob& J, const double* F1, int ld1, int mo, int q0, int kc, int orow, int ocol,
                           int j0, int wc, double* S, const double* Ts) {
  const int tid = threadIdx.x;
  const int kcp = (kc + 3) & ~3;
  for (int i0 = 0; i0 < mo; i0 += kT) {
    const int mc = min(kT, mo - i0);
    double old[WarpTiling<8, NCT>::RTW * WarpTiling<8, NCT>::CTW][2];
    load_out<NCT>(J, orow, ocol, i0, mc, j0, wc, old);
    for (int e = tid; e < kT * kcp; e += kNT) {   // S[i + q * 68] = F1(i0 + i, q0 + q)
      const int i = e & (kT - 1), q = e >> 6;
      if (i >= mc) continue;
      const bool ok = q < kc;
      cp8(S + i + q * kLd, ok ? F1 + (i0 + i) + (int64_t)(q0 + q) * ld1 : F1, ok);
    }
    cp_wait();
    __syncthreads();
    double acc[WarpTiling<8, NCT>::RTW * WarpTiling<8, NCT>::CTW][2];
    acc_zero<8, NCT>(acc);
    tile_dmma<8, NCT>(S, 1, kLd, Ts, kLdJ, 1, (kc + 3) & ~3, acc);
    store_acc_old<NCT>(J, orow, ocol, i0, mc, j0, wc, acc, old);
    __syncthreads();
  }
}

__device__ void apply_f1(const EvalJob& J, const double* F1, int ld1, int mo, int q0, int kc, int orow, int ocol,
                         int j0, int wc, double* S, const double* Ts) {
  if (wc <= 8) apply_f1_t<1>(J, F1, ld1, mo, q0, kc, orow, ocol, j0, wc, S, Ts);
  else if (wc <= 16) apply_f1_t<2>(J, F1, ld1, mo, q0, kc, orow, ocol, j0, wc, S, Ts);
  else apply_f1_t<4>(J, F1, ld1, mo, q0, kc, orow, ocol, j0, wc, S, Ts);
}

// Ts(q, j) = sum_p F2(p, q0 + q) V(vrow + p, j0 + j)  (q < 32, j < 8 NCT), by DMMA
// over 64-row chunks of F2 (staged p-contiguous: S[p + q * 68])
template <int NCT>
__device__ void lowrank_t(const EvalJob& J, const double* F2, int ld2, int ko, int vrow, int q0, int kc, int j0,
                          int wc, double* S, double* Vs, double* Ts) {
  using WT = WarpTiling<4, NCT>;
  const int tid = threadIdx.x;
  double acc[WT::RTW * WT::CTW][2];
  acc_zero<4, NCT>(acc);
  const int kcp = (kc + 3) & ~3;   // T rows [kc, kcp) are zero; rows >= kcp are never read
  for (int p0 = 0; p0 < ko; p0 += kT) {
    const int pc = min(kT, ko - p0), pcp = (pc + 3) & ~3;
    for (int e = tid; e < kT * kcp; e += kNT) {
      const int p = e & (kT - 1), q = e >> 6;
      if (p >= pcp) continue;
      const bool ok = p < pc && q < kc;
      cp8(S + p + q * kLd, ok ? F2 + (p0 + p) + (int64_t)(q0 + q) * ld2 : F2, ok);
    }
    int brs, bcs;
    stage_v(J, vrow, p0, pc, j0, wc, Vs, brs, bcs);
    cp_wait();
    __syncthreads();
    tile_dmma<4, NCT>(S, kLd, 1, Vs, brs, bcs, (pc + 3) & ~3, acc);
    __syncthreads();
  }
  // fragments -> Ts (every (q, j) of the 32 x 8 NCT tile is written; q >= kc rows are 0)
  const int lane = tid & 31, warp = tid >> 5;
  if (warp < WT::RG * WT::CG) {
    const int rg = warp % WT::RG, cg = warp / WT::RG;
#pragma unroll
    for (int r = 0; r < WT::RTW; r++)
#pragma unroll
      for (int c = 0; c < WT::CTW; c++) {
        const int q = (rg * WT::RTW + r) * 8 + (lane >> 2);
        const int j = (cg * WT::CTW + c) * 8 + 2 * (lane & 3);
        Ts[j + q * kLdJ] = acc[r * WT::CTW + c][0];
        Ts[j + 1 + q * kLdJ] = acc[r * WT::CTW + c][1];
      }
  }
  __syncthreads();
}

__device__ void eval_lowrank(const EvalJob& J, const LeafDesc& L, int orow, int vrow, int mo, int ko, double* S,
                             double* Vs, double* Ts) {
  const double* F1 = J.trans ? L.B : L.A;
  const int ld1 = J.trans ? L.n : L.m;
  const double* F2 = J.trans ? L.A : L.B;
  const int ld2 = J.trans ? L.m : L.n;
  for (int j0 = 0; j0 < J.w; j0 += kW) {
    const int wc = min(kW, J.w - j0);
    for (int q0 = 0; q0 < L.k; q0 += kW) {
      const int kc = min(kW, L.k - q0);
      if (wc <= 8) lowrank_t<1>(J, F2, ld2, ko, vrow, q0, kc, j0, wc, S, Vs, Ts);
      else if (wc <= 16) lowrank_t<2>(J, F2, ld2, ko, vrow, q0, kc, j0, wc, S, Vs, Ts);
      else lowrank_t<4>(J, F2, ld2, ko, vrow, q0, kc, j0, wc, S, Vs, Ts);
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
      const int kcp = (kc + 3) & ~3;
      for (int e = tid; e < kW * kcp; e += kNT) {   // Ts(q, j) = F2(j0 + j, q0 + q) at j + q * 36
        const int j = e & (kW - 1), q = e >> 5;
        if (j >= wc) continue;
        const bool ok = q < kc;
        cp8(Ts + j + q * kLdJ, ok ? F2 + (j0 + j) + (int64_t)(q0 + q) * ld2 : F2, ok);
      }
      cp_wait();
      __syncthreads();
      apply_f1(J, F1, ld1, mo, q0, kc, orow, vrow, j0, wc, S, Ts);
    }
  }
}
}  // namespace

__device__ void eval_range(const EvalJob& J, int lb, int le, double* sm) {
  double* S = sm;
  double* Vt = S + kSmemS;
  double* Ts = Vt + kSmemV;
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

__global__ void __launch_bounds__(kNT, 3) k_eval2(const EvalJob* __restrict__ jobs) {
  extern __shared__ double sm[];
  const EvalJob* jp = &jobs[blockIdx.x];
  while (jp) {
    const EvalJob J = *jp;
    if (J.nrng == 0) {
      eval_range(J, J.leaf_begin, J.leaf_end, sm);
    } else {
      for (int g = 0; g < J.nrng; g++) {
        const int2 r = J.rng[g];
        eval_range(J, r.x, r.y, sm);
      }
    }
    jp = J.next;   // eval_range ends with a barrier: the chained job sees this one's writes
  }
}

// ------------------------------------------------------------------ GEMM
// C = alpha op(A) op(B) + beta C on the FP64 tensor pipe: one 64 x 64 output
// tile per CTA (host tile map), K chunks of 16 staged by cp.async in the
// orientation that keeps both the global loads coalesced and the DMMA
// fragment loads conflict-free (leading dimensions 68 / 20 = 4 mod 16);
// warp (rg, cg) owns rows 16 rg .. +16 and columns 32 cg .. +32 (2 x 4 tiles).
// Stored-upper masks (R factors sharing storage with reflectors) read as 0.
__global__ void __launch_bounds__(256) k_gemm2(const GemmJob* __restrict__ jobs, const int* __restrict__ tmap) {
  __shared__ __align__(16) double As[64 * 20];
  __shared__ __align__(16) double Bs[64 * 20];
  const int64_t tile = blockIdx.x;
  const GemmJob& J = jobs[tmap[tile]];
  const int m = J.m;
  const int n = J.ndyn ? *J.ndyn : J.n;
  const int k = J.kdyn ? *J.kdyn : J.k;
  const int mt = (m + 63) >> 6;
  const int64_t local = tile - J.tile0;
  const int ti = (int)(local % mt), tj = (int)(local / mt);
  if (tj * 64 >= n || ti * 64 >= m) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int lr = lane >> 2, lk = lane & 3, rg = warp & 3, cg = warp >> 2;
  const int ars = J.transA ? 20 : 1, acs = J.transA ? 1 : kLd;
  const int brs = J.transB ? kLd : 1, bcs = J.transB ? 1 : 20;
  double acc[2][4][2];
#pragma unroll
  for (int r = 0; r < 2; r++)
#pragma unroll
    for (int c = 0; c < 4; c++) acc[r][c][0] = acc[r][c][1] = 0.0;
  for (int p0 = 0; p0 < k; p0 += 16) {
    for (int e = tid; e < 1024; e += 256) {
      int i, p;
      double* dst;
      if (!J.transA) { i = e & 63; p = e >> 6; dst = As + i + p * kLd; }
      else { p = e & 15; i = e >> 4; dst = As + p + i * 20; }
      const int gi = ti * 64 + i, gp = p0 + p;
      const int r = J.transA ? gp : gi, c = J.transA ? gi : gp;
      const bool ok = gi < m && gp < k && !(J.maskA && r > c);
      cp8(dst, ok ? J.A + r + (int64_t)c * J.lda : J.A, ok);
    }
    for (int e = tid; e < 1024; e += 256) {
      int j, p;
      double* dst;
      if (J.transB) { j = e & 63; p = e >> 6; dst = Bs + j + p * kLd; }
      else { p = e & 15; j = e >> 4; dst = Bs + p + j * 20; }
      const int gj = tj * 64 + j, gp = p0 + p;
      const int r = J.transB ? gj : gp, c = J.transB ? gp : gj;
      const bool ok = gj < n && gp < k && !(J.maskB && r > c);
      cp8(dst, ok ? J.B + r + (int64_t)c * J.ldb : J.B, ok);
    }
    cp_wait();
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; kk += 4) {
      double a[2], b[4];
#pragma unroll
      for (int r = 0; r < 2; r++) a[r] = As[(rg * 16 + r * 8 + lr) * ars + (kk + lk) * acs];
#pragma unroll
      for (int c = 0; c < 4; c++) b[c] = Bs[(kk + lk) * brs + (cg * 32 + c * 8 + lr) * bcs];
#pragma unroll
      for (int r = 0; r < 2; r++)
#pragma unroll
        for (int c = 0; c < 4; c++) dmma(acc[r][c], a[r], b[c]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < 2; r++) {
    const int gi = ti * 64 + rg * 16 + r * 8 + lr;
    if (gi >= m) continue;
#pragma unroll
    for (int c = 0; c < 4; c++)
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int gj = tj * 64 + cg * 32 + c * 8 + 2 * lk + h;
        if (gj >= n) continue;
        double* d = J.C + gi + (int64_t)gj * J.ldc;
        const double v = J.alpha * acc[r][c][h];
        *d = (J.beta == 0.0) ? v : fma(J.beta, *d, v);
      }
  }
}

void launch_gemm2(const GemmJob* d_jobs, const int* d_tmap, int64_t ntiles, cudaStream_t st) {
  k_gemm2<<<(unsigned)ntiles, 256, 0, st>>>(d_jobs, d_tmap);
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
      const int mm = S.m;
      // reversed (upper) steps: row i of the forward sweep is row mm-1-i of T / the panel
      auto tr_at = [&](int i, int p) {
        const int a = S.rev ? mm - 1 - i : i, b = S.rev ? mm - 1 - p : p;
        return S.trans ? S.P[b + (int64_t)a * S.ld] : S.P[a + (int64_t)b * S.ld];
      };
      for (int col = tid; col < J.ncols; col += kNT) {
        double* x = v + (int64_t)col * J.ldv;
        for (int i = 0; i < mm; i++) {
          const int xi = S.rev ? mm - 1 - i : i;
          double acc = x[xi];
          for (int p = 0; p < i; p++) acc = fma(-tr_at(i, p), x[S.rev ? mm - 1 - p : p], acc);
          x[xi] = S.unit ? acc : acc / tr_at(i, i);
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
        const int a = S.rev ? m - 1 - i : i, b = S.rev ? m - 1 - j : j;
        tri[i + j * kLdS] = S.trans ? S.P[b + (int64_t)a * S.ld] : S.P[a + (int64_t)b * S.ld];
      }
      __syncthreads();
      for (int i = tid; i < m; i += kNT) dinv[i] = S.unit ? 1.0 : 1.0 / tri[i + i * kLdS];
      const int ldx = m + 1;
      for (int c0 = 0; c0 < J.ncols; c0 += kTrsmCols) {
        const int cc = min(kTrsmCols, J.ncols - c0);
        for (int e = tid; e < m * cc; e += kNT) {
          const int i = e % m, c = e / m;
          xs[c * ldx + i] = v[(S.rev ? m - 1 - i : i) + (int64_t)(c0 + c) * J.ldv];
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
          v[(S.rev ? m - 1 - i : i) + (int64_t)(c0 + c) * J.ldv] = xs[c * ldx + i] * dinv[i];
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
  ensure_smem_attr((const void*)k_trsm2, kTrsmShared * 8);
  count_launch();
  k_trsm2<<<njobs, kNT, (size_t)kTrsmShared * 8, st>>>(d_jobs, d_steps, leaves);
}

void launch_eval2(const EvalJob* d_jobs, int njobs, cudaStream_t st) {
  if (njobs <= 0) return;
  ensure_smem_attr((const void*)k_eval2, kSmem * 8);
  count_launch();
  k_eval2<<<njobs, kNT, (size_t)kSmem * 8, st>>>(d_jobs);
}

}  // namespace hm
