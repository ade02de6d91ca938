// Batched FP64 kernels of libhm (sm_100a).
//
// FP64 on B200 runs on the DFMA pipe (mma.sync f64 lowers to DMMA 8x8x4 with
// the same peak; tcgen05 has no f64 kind -- DESIGN.md §5).  All kernels are
// "one job list per launch": a device array of heterogeneous job
// descriptors, one CTA (or a tile range) per job, so one launch covers a
// whole level of the block tree (Parallelization remark).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <atomic>
#include <mutex>
#include <set>
#include <stdexcept>
#include <string>
#include <tuple>

#include <cstdlib>

#include "kernels.h"

namespace hm {

static constexpr double kU = 1.1102230246251565e-16;  // unit roundoff 2^-53

static std::atomic<long long> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

void ensure_smem_attr(const void* func, int bytes) {
  static std::mutex mu;
  static std::set<std::tuple<const void*, int, int>> done;   // (function, device, bytes)
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  const auto key = std::make_tuple(func, dev, bytes);
  if (done.count(key)) return;
  const cudaError_t e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw std::runtime_error(std::string("cudaFuncSetAttribute(MaxDynamicSharedMemorySize): ") + cudaGetErrorString(e));
  }
  done.insert(key);
}
int64_t launch_count() { return g_launches.load(); }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide sum for blockDim.x == 256; result broadcast to all threads.
__device__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x < 32) {
    s = (lane < (int)(blockDim.x >> 5)) ? red[lane] : 0.0;
    s = warp_sum(s);
    if (lane == 0) red[0] = s;
  }
  __syncthreads();
  s = red[0];
  __syncthreads();
  return s;
}

template <class J>
__device__ __forceinline__ int find_job(const J* jobs, int njobs, int64_t tile) {
  int lo = 0, hi = njobs - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (jobs[mid].tile0 <= tile) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// ------------------------------------------------------------------ GEMM
// 64x64 output tile per CTA, K chunks of 16, 256 threads x (4x4) outputs.
__global__ void __launch_bounds__(256) k_gemm(const GemmJob* __restrict__ jobs, int njobs, const int* __restrict__ tmap) {
  __shared__ double As[16][64 + 1];
  __shared__ double Bs[16][64 + 1];
  const int64_t tile = blockIdx.x;
  const GemmJob& J = jobs[tmap ? tmap[tile] : find_job(jobs, njobs, tile)];
  const int m = J.m;
  const int n = J.ndyn ? *J.ndyn : J.n;
  const int k = J.kdyn ? *J.kdyn : J.k;
  const int mt = (m + 63) >> 6;
  const int64_t local = tile - J.tile0;
  const int ti = (int)(local % mt), tj = (int)(local / mt);
  if (tj * 64 >= n || ti * 64 >= m) return;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; a++)
#pragma unroll
    for (int b = 0; b < 4; b++) acc[a][b] = 0.0;
  for (int p0 = 0; p0 < k; p0 += 16) {
    for (int e = threadIdx.x; e < 1024; e += 256) {
      int i, p;
      if (!J.transA) { i = e & 63; p = e >> 6; } else { p = e & 15; i = e >> 4; }
      const int gi = ti * 64 + i, gp = p0 + p;
      double v = 0.0;
      if (gi < m && gp < k) {
        const int r = J.transA ? gp : gi, c = J.transA ? gi : gp;
        if (!(J.maskA && r > c)) v = J.A[r + (int64_t)c * J.lda];
      }
      As[p][i] = v;
    }
    for (int e = threadIdx.x; e < 1024; e += 256) {
      int j, p;
      if (!J.transB) { p = e & 15; j = e >> 4; } else { j = e & 63; p = e >> 6; }
      const int gj = tj * 64 + j, gp = p0 + p;
      double v = 0.0;
      if (gj < n && gp < k) {
        const int r = J.transB ? gj : gp, c = J.transB ? gp : gj;
        if (!(J.maskB && r > c)) v = J.B[r + (int64_t)c * J.ldb];
      }
      Bs[p][j] = v;
    }
    __syncthreads();
#pragma unroll
    for (int p = 0; p < 16; p++) {
      double a[4], b[4];
#pragma unroll
      for (int q = 0; q < 4; q++) { a[q] = As[p][tx + 16 * q]; b[q] = Bs[p][ty + 16 * q]; }
#pragma unroll
      for (int x = 0; x < 4; x++)
#pragma unroll
        for (int y = 0; y < 4; y++) acc[x][y] = fma(a[x], b[y], acc[x][y]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int y = 0; y < 4; y++) {
    const int gj = tj * 64 + ty + 16 * y;
    if (gj >= n) continue;
#pragma unroll
    for (int x = 0; x < 4; x++) {
      const int gi = ti * 64 + tx + 16 * x;
      if (gi >= m) continue;
      double* c = J.C + gi + (int64_t)gj * J.ldc;
      const double v = J.alpha * acc[x][y];
      *c = (J.beta == 0.0) ? v : fma(J.beta, *c, v);
    }
  }
}

void launch_gemm(const GemmJob* d_jobs, int njobs, int64_t ntiles, cudaStream_t st) {
  if (njobs <= 0 || ntiles <= 0) return;
  count_launch();
  k_gemm<<<(unsigned)ntiles, 256, 0, st>>>(d_jobs, njobs, nullptr);
}

void launch_gemm2(const GemmJob* d_jobs, const int* d_tmap, int64_t ntiles, cudaStream_t st);   // eval.cu (DMMA)

void launch_gemm_mapped(const GemmJob* d_jobs, int njobs, const int* d_tmap, int64_t ntiles, cudaStream_t st) {
  if (njobs <= 0 || ntiles <= 0) return;
  count_launch();
  static const bool old = std::getenv("HM_GEMM_OLD") != nullptr;
  if (old || !d_tmap) k_gemm<<<(unsigned)ntiles, 256, 0, st>>>(d_jobs, njobs, d_tmap);
  else launch_gemm2(d_jobs, d_tmap, ntiles, st);
}

// ------------------------------------------------------------------ QR
// Householder QR (dgeqr2) of one tall panel per CTA; in shared memory when
// m*n <= cap, else in place in global memory.
__global__ void __launch_bounds__(256) k_qr(const QrJob* __restrict__ jobs, int cap) {
  extern __shared__ double sm[];
  __shared__ double red[32];
  __shared__ double s_tau, s_scale;
  const QrJob J = jobs[blockIdx.x];
  const int m = J.m, n = J.n;
  const bool use_sm = (int64_t)m * n <= cap;
  double* A = use_sm ? sm : J.A;
  const int lda = use_sm ? m : J.lda;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (use_sm) {
    for (int64_t e = tid; e < (int64_t)m * n; e += 256) {
      const int i = (int)(e % m), c = (int)(e / m);
      sm[e] = J.A[i + (int64_t)c * J.lda];
    }
    __syncthreads();
  }
  for (int j = 0; j < n; j++) {
    double* x = A + (int64_t)j * lda;
    double part = 0.0;
    for (int i = j + 1 + tid; i < m; i += 256) part += x[i] * x[i];
    const double xn2 = block_sum(part, red);
    if (tid == 0) {
      const double alpha = x[j];
      double tau = 0.0, scale = 0.0, beta = alpha;
      if (xn2 > 0.0) {
        beta = -copysign(sqrt(alpha * alpha + xn2), alpha);
        tau = (beta - alpha) / beta;
        scale = 1.0 / (alpha - beta);
      }
      x[j] = beta;
      J.tau[j] = tau;
      s_tau = tau;
      s_scale = scale;
    }
    __syncthreads();
    const double tau = s_tau, scale = s_scale;
    if (tau != 0.0)
      for (int i = j + 1 + tid; i < m; i += 256) x[i] *= scale;
    __syncthreads();
    if (tau != 0.0) {
      for (int c = j + 1 + warp; c < n; c += 8) {
        double* y = A + (int64_t)c * lda;
        double s = 0.0;
        for (int i = j + 1 + lane; i < m; i += 32) s += x[i] * y[i];
        s = warp_sum(s) + y[j];
        s *= tau;
        if (lane == 0) y[j] -= s;
        for (int i = j + 1 + lane; i < m; i += 32) y[i] -= s * x[i];
      }
    }
    __syncthreads();
  }
  if (use_sm) {
    for (int64_t e = tid; e < (int64_t)m * n; e += 256) {
      const int i = (int)(e % m), c = (int)(e / m);
      J.A[i + (int64_t)c * J.lda] = sm[e];
    }
  }
}

int qr_smem_capacity() { return 24 * 1024; }

void launch_qr(const QrJob* d_jobs, int njobs, int cap, cudaStream_t st) {
  if (njobs <= 0) return;
  if (cap > qr_smem_capacity()) cap = qr_smem_capacity();
  const size_t bytes = (size_t)cap * sizeof(double);
  ensure_smem_attr((const void*)k_qr, qr_smem_capacity() * 8);
  count_launch();
  k_qr<<<njobs, 256, bytes, st>>>(d_jobs, cap);
}

// ------------------------------------------------------------------ apply Q
// X <- H_0 ... H_{r-1} X ; one warp per column of X (grid.y spreads the
// columns over CTAs), reflectors read from L2.  With the QR's compact-WY T
// factors the reflectors are applied 16 at a time (Q_p = I - Y_p T_p Y_p^T,
// last panel first): two passes over the rows per panel instead of two per
// reflector.
__global__ void __launch_bounds__(256, 3) k_applyq(const ApplyQJob* __restrict__ jobs) {
  const ApplyQJob J = jobs[blockIdx.x];
  const int c = J.cdyn ? *J.cdyn : J.c;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int col = blockIdx.y * 8 + warp;
  if (col >= c) return;
  double* x = J.X + (int64_t)col * J.ldx;
  if (J.T) {
    for (int p = (J.r + 15) / 16 - 1; p >= 0; p--) {
      const int j0 = p * 16, kb = min(16, J.r - j0);
      const double* Vp = J.V + (int64_t)j0 * J.ldv;
      double w[16];
#pragma unroll
      for (int q = 0; q < 16; q++) w[q] = 0.0;
      // the 16 reflector rows beyond the panel's unit triangle, 2 rows per
      // lane per step (34 loads in flight)
      int i = j0 + lane;
      for (; i < j0 + 16 && i < J.m; i += 32) {
        const double xi = x[i];
#pragma unroll
        for (int q = 0; q < 16; q++)
          if (q < kb) {
            const double y = i > j0 + q ? Vp[i + (int64_t)q * J.ldv] : (i == j0 + q ? 1.0 : 0.0);
            w[q] = fma(y, xi, w[q]);
          }
      }
      for (; i + 32 < J.m; i += 64) {
        const double xa = x[i], xb = x[i + 32];
#pragma unroll
        for (int q = 0; q < 16; q++)
          if (q < kb) w[q] = fma(Vp[i + 32 + (int64_t)q * J.ldv], xb, fma(Vp[i + (int64_t)q * J.ldv], xa, w[q]));
      }
      for (; i < J.m; i += 32) {
        const double xi = x[i];
#pragma unroll
        for (int q = 0; q < 16; q++)
          if (q < kb) w[q] = fma(Vp[i + (int64_t)q * J.ldv], xi, w[q]);
      }
#pragma unroll
      for (int q = 0; q < 16; q++) w[q] = warp_sum(w[q]);
      const double* Tp = J.T + 256 * p;
      double z[16];
#pragma unroll
      for (int q = 0; q < 16; q++) {
        double s = 0.0;
#pragma unroll
        for (int r = q; r < 16; r++)
          if (r < kb) s = fma(Tp[q + r * 16], w[r], s);
        z[q] = s;
      }
      i = j0 + lane;
      for (; i < j0 + 16 && i < J.m; i += 32) {
        double s = 0.0;
#pragma unroll
        for (int q = 0; q < 16; q++)
          if (q < kb) {
            const double y = i > j0 + q ? Vp[i + (int64_t)q * J.ldv] : (i == j0 + q ? 1.0 : 0.0);
            s = fma(y, z[q], s);
          }
        x[i] -= s;
      }
      for (; i + 32 < J.m; i += 64) {
        const double xa = x[i], xb = x[i + 32];
        double sa = 0.0, sb = 0.0;
#pragma unroll
        for (int q = 0; q < 16; q++)
          if (q < kb) {
            sa = fma(Vp[i + (int64_t)q * J.ldv], z[q], sa);
            sb = fma(Vp[i + 32 + (int64_t)q * J.ldv], z[q], sb);
          }
        x[i] = xa - sa;
        x[i + 32] = xb - sb;
      }
      for (; i < J.m; i += 32) {
        double s = 0.0;
#pragma unroll
        for (int q = 0; q < 16; q++)
          if (q < kb) s = fma(Vp[i + (int64_t)q * J.ldv], z[q], s);
        x[i] -= s;
      }
      __syncwarp();
    }
    return;
  }
  for (int j = J.r - 1; j >= 0; j--) {
    const double tau = J.tau[j];
    if (tau == 0.0) continue;
    const double* v = J.V + (int64_t)j * J.ldv;
    double s = 0.0;
    for (int i = j + 1 + lane; i < J.m; i += 32) s += v[i] * x[i];
    s = (warp_sum(s) + x[j]) * tau;
    if (lane == 0) x[j] -= s;
    for (int i = j + 1 + lane; i < J.m; i += 32) x[i] -= s * v[i];
    __syncwarp();
  }
}

void launch_applyq(const ApplyQJob* d_jobs, int njobs, int cmax, cudaStream_t st) {
  if (njobs <= 0 || cmax <= 0) return;
  count_launch();
  k_applyq<<<dim3(njobs, (cmax + 7) / 8), 256, 0, st>>>(d_jobs);
}

// SVD kernels: see svd.cu

// ------------------------------------------------------------------ copy
// tmap (optional): job index of every tile (host-built; one load instead of a
// binary search of dependent loads per CTA)
__global__ void __launch_bounds__(256) k_copy(const CopyJob* __restrict__ jobs, int njobs, const int* __restrict__ tmap) {
  const int64_t tile = blockIdx.x;
  const CopyJob& J = jobs[tmap ? tmap[tile] : find_job(jobs, njobs, tile)];
  const int mt = (J.rows + 31) >> 5;
  const int64_t local = tile - J.tile0;
  const int ti = (int)(local % mt), tj = (int)(local / mt);
  for (int e = threadIdx.x; e < 1024; e += 256) {
    const int i = ti * 32 + (e & 31), j = tj * 32 + (e >> 5);
    if (i >= J.rows || j >= J.cols) continue;
    double v;
    if (J.identity) {
      if (i != j) continue;
      v = J.coef;
    } else if (J.upper && i > j) {
      v = 0.0;
    } else {
      v = J.coef * (J.trans ? J.src[j + (int64_t)i * J.lds] : J.src[i + (int64_t)j * J.lds]);
    }
    double* d = J.dst + i + (int64_t)j * J.ldd;
    *d = J.accumulate ? (*d + v) : v;
  }
}

void launch_copy(const CopyJob* d_jobs, int njobs, int64_t ntiles, cudaStream_t st) {
  if (njobs <= 0 || ntiles <= 0) return;
  count_launch();
  k_copy<<<(unsigned)ntiles, 256, 0, st>>>(d_jobs, njobs, nullptr);
}

void launch_copy_mapped(const CopyJob* d_jobs, int njobs, const int* d_tmap, int64_t ntiles, cudaStream_t st) {
  if (njobs <= 0 || ntiles <= 0) return;
  count_launch();
  k_copy<<<(unsigned)ntiles, 256, 0, st>>>(d_jobs, njobs, d_tmap);
}

// ------------------------------------------------------------------ eval
// ------------------------------------------------------------------ dense leaf factorizations
// In-place LU without pivoting (unit L) or Cholesky (lower) of one diagonal
// leaf per CTA (m <= 128 in shared memory).  Pivot breakdown (|p| <= 1e-300,
// non-finite, or a non-positive Cholesky pivot) sets *fail = cluster id + 1
// (first failure wins); minpiv[job] = min |pivot|.
__global__ void __launch_bounds__(256) k_leaf_factor(const LeafFactorJob* __restrict__ jobs, int chol,
                                                     int* fail, double* minpiv) {
  extern __shared__ double a[];
  __shared__ double s_piv;
  const LeafFactorJob J = jobs[blockIdx.x];
  const int m = J.m, tid = threadIdx.x;
  for (int e = tid; e < m * m; e += blockDim.x) a[e] = J.N[(e % m) + (int64_t)(e / m) * J.ld];
  __syncthreads();
  double mp = 1e300;
  bool bad = false;
  for (int j = 0; j < m; j++) {
    if (tid == 0) {
      double p = a[j + j * m];
      if (chol) {
        p = (p > 0.0 && isfinite(p)) ? sqrt(p) : -1.0;
        if (p > 0.0) a[j + j * m] = p;
      }
      s_piv = p;
    }
    __syncthreads();
    const double p = s_piv;
    if (!isfinite(p) || fabs(p) <= 1e-300 || (chol && p <= 0.0)) { bad = true; break; }
    mp = fmin(mp, fabs(p));
    for (int i = j + 1 + tid; i < m; i += blockDim.x) a[i + j * m] /= p;
    __syncthreads();
    // trailing update: lower-right block (Cholesky: lower triangle only)
    const int r = m - j - 1;
    for (int e = tid; e < r * r; e += blockDim.x) {
      const int i = j + 1 + e % r, c = j + 1 + e / r;
      if (chol && c > i) continue;
      a[i + c * m] -= a[i + j * m] * (chol ? a[c + j * m] : a[j + c * m]);
    }
    __syncthreads();
  }
  if (bad) {
    if (tid == 0) atomicCAS(fail, 0, J.cluster + 1);
    return;
  }
  for (int e = tid; e < m * m; e += blockDim.x) {
    const int i = e % m, c = e / m;
    J.N[i + (int64_t)c * J.ld] = (chol && c > i) ? 0.0 : a[e];
  }
  if (tid == 0 && minpiv) minpiv[blockIdx.x] = mp;
}

// In-place inverse of one diagonal leaf per CTA by Gauss-Jordan elimination
// without pivoting ("standard linear algebra"; the
// paper assumes every principal submatrix invertible).  Pivot
// breakdown sets *fail = cluster id + 1; minpiv[job] = min |pivot|.
__global__ void __launch_bounds__(256) k_leaf_inverse(const LeafFactorJob* __restrict__ jobs, int* fail,
                                                      double* minpiv) {
  extern __shared__ double a[];
  double* f = a + (size_t)jobs[blockIdx.x].m * jobs[blockIdx.x].m;
  __shared__ double s_piv;
  const LeafFactorJob J = jobs[blockIdx.x];
  const int m = J.m, tid = threadIdx.x;
  for (int e = tid; e < m * m; e += blockDim.x) a[e] = J.N[(e % m) + (int64_t)(e / m) * J.ld];
  __syncthreads();
  double mp = 1e300;
  for (int k = 0; k < m; k++) {
    if (tid == 0) s_piv = a[k + k * m];
    for (int i = tid; i < m; i += blockDim.x) f[i] = a[i + k * m];   // column k before the step
    __syncthreads();
    const double p = s_piv;
    if (!isfinite(p) || fabs(p) <= 1e-300) {
      if (tid == 0) atomicCAS(fail, 0, J.cluster + 1);
      return;
    }
    mp = fmin(mp, fabs(p));
    const double pinv = 1.0 / p;
    // row k: A[k][j] /= p (j != k), A[k][k] = 1/p
    for (int j = tid; j < m; j += blockDim.x) a[k + j * m] = (j == k ? 1.0 : a[k + j * m]) * pinv;
    __syncthreads();
    // rows i != k: A[i][j] -= f_i A[k][j] (j != k), A[i][k] = -f_i / p
    for (int e = tid; e < m * m; e += blockDim.x) {
      const int i = e % m, j = e / m;
      if (i == k) continue;
      a[e] = (j == k ? 0.0 : a[e]) - f[i] * a[k + j * m];
    }
    __syncthreads();
  }
  for (int e = tid; e < m * m; e += blockDim.x) J.N[(e % m) + (int64_t)(e / m) * J.ld] = a[e];
  if (tid == 0 && minpiv) minpiv[blockIdx.x] = mp;
}

void launch_leaf_inverse(const LeafFactorJob* d_jobs, int njobs, int* fail, double* minpiv, int maxm,
                         cudaStream_t st) {
  if (njobs <= 0) return;
  ensure_smem_attr((const void*)k_leaf_inverse, 210 * 1024);
  count_launch();
  k_leaf_inverse<<<njobs, 256, (size_t)maxm * (maxm + 1) * 8, st>>>(d_jobs, fail, minpiv);
}

// table[patch[i].pos] = patch[i].leaf: the leaf descriptors of the blocks one
// flush has rewritten, in ONE launch (instead of one H2D copy per block)
__global__ void k_patch_leaves(LeafDesc* __restrict__ table, const LeafPatch* __restrict__ patch, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) table[patch[i].pos] = patch[i].leaf;
}

void launch_patch_leaves(LeafDesc* table, const LeafPatch* d_patch, int n, cudaStream_t st) {
  if (n <= 0) return;
  count_launch();
  k_patch_leaves<<<(n + 127) / 128, 128, 0, st>>>(table, d_patch, n);
}

// dst_i[0:count_i] = 0 for a list of device ranges (zeroing H-matrix blocks)
__global__ void k_zero_ranges(double* const* __restrict__ ptr, const int64_t* __restrict__ cnt) {
  double* p = ptr[blockIdx.x];
  const int64_t n = cnt[blockIdx.x];
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) p[i] = 0.0;
}

void launch_zero_ranges(double* const* d_ptr, const int64_t* d_cnt, int n, cudaStream_t st) {
  if (n <= 0) return;
  count_launch();
  k_zero_ranges<<<n, 256, 0, st>>>(d_ptr, d_cnt);
}

void launch_leaf_factor(const LeafFactorJob* d_jobs, int njobs, int chol, int* fail, double* minpiv,
                        int maxm, cudaStream_t st) {
  if (njobs <= 0) return;
  ensure_smem_attr((const void*)k_leaf_factor, 200 * 1024);
  count_launch();
  k_leaf_factor<<<njobs, 256, (size_t)maxm * maxm * 8, st>>>(d_jobs, chol, fail, minpiv);
}

// ------------------------------------------------------------------ entries
// G_ij = w_j / (4 pi |x_i - x_j|), G_ii = sqrt(w_i/pi)/2 (BASELINE.json),
// evaluated with explicit round-to-nearest ops (no FMA contraction).
__device__ __forceinline__ double g_slp(const double* x, const double* w, int64_t i, int64_t j) {
  if (i == j) return __dmul_rn(__dsqrt_rn(__ddiv_rn(w[i], M_PI)), 0.5);
  const double dx = __dsub_rn(x[3 * i], x[3 * j]);
  const double dy = __dsub_rn(x[3 * i + 1], x[3 * j + 1]);
  const double dz = __dsub_rn(x[3 * i + 2], x[3 * j + 2]);
  const double r2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
  return __ddiv_rn(w[j], __dmul_rn(4.0 * M_PI, __dsqrt_rn(r2)));
}

// K_ij = w_j ((x_j - x_i) . n_j) / (4 pi |x_i - x_j|^3), K_ii = 1/2: the
// double layer + 1/2 I (sign reading R20), same
// operation order as oracle/kernel.py dlp_entries.
__device__ __forceinline__ double g_dlp(const double* x, const double* w, const double* nr, int64_t i, int64_t j) {
  if (i == j) return 0.5;
  const double dx = __dsub_rn(x[3 * j], x[3 * i]);
  const double dy = __dsub_rn(x[3 * j + 1], x[3 * i + 1]);
  const double dz = __dsub_rn(x[3 * j + 2], x[3 * i + 2]);
  const double dot = __dadd_rn(__dadd_rn(__dmul_rn(dx, nr[3 * j]), __dmul_rn(dy, nr[3 * j + 1])), __dmul_rn(dz, nr[3 * j + 2]));
  const double r2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
  const double r = __dsqrt_rn(r2);
  return __ddiv_rn(__dmul_rn(w[j], dot), __dmul_rn(__dmul_rn(4.0 * M_PI, r2), r));
}

__global__ void __launch_bounds__(256) k_gen(const GenJob* __restrict__ jobs, int njobs,
                                             const double* __restrict__ x,
                                             const double* __restrict__ w,
                                             const double* __restrict__ nr,
                                             const int64_t* __restrict__ perm, int kernel) {
  const int64_t tile = blockIdx.x;
  const GenJob& J = jobs[find_job(jobs, njobs, tile)];
  const int mt = (J.m + 31) >> 5;
  const int64_t local = tile - J.tile0;
  const int ti = (int)(local % mt), tj = (int)(local / mt);
  for (int e = threadIdx.x; e < 1024; e += 256) {
    const int i = ti * 32 + (e & 31), j = tj * 32 + (e >> 5);
    if (i >= J.m || j >= J.n) continue;
    const int64_t oi = perm[J.r0 + i], oj = perm[J.c0 + j];
    double v;
    if (kernel == 2) {
      v = g_dlp(x, w, nr, oi, oj);
    } else {
      v = g_slp(x, w, oi, oj);
      if (kernel == 1) v = __dmul_rn(0.5, __dadd_rn(v, g_slp(x, w, oj, oi)));
    }
    J.dst[i + (int64_t)j * J.ld] = v;
  }
}

void launch_gen(const GenJob* d_jobs, int njobs, int64_t ntiles, const double* x, const double* w,
                const double* nrm, const int64_t* perm, int kernel, cudaStream_t st) {
  if (njobs <= 0 || ntiles <= 0) return;
  count_launch();
  k_gen<<<(unsigned)ntiles, 256, 0, st>>>(d_jobs, njobs, x, w, nrm, perm, kernel);
}

// ------------------------------------------------------------------ norms
__global__ void __launch_bounds__(256) k_norm(const NormJob* __restrict__ jobs, double* out) {
  __shared__ double red[32];
  const NormJob J = jobs[blockIdx.x];
  const int n = J.ndyn ? *J.ndyn : J.n;
  double s = 0.0;
  for (int64_t e = threadIdx.x; e < (int64_t)J.m * n; e += 256) {
    const double v = J.A[(e % J.m) + (e / J.m) * J.lda];
    s = fma(v, v, s);
  }
  s = block_sum(s, red);
  if (threadIdx.x == 0) out[blockIdx.x] = s;
}

void launch_norm(const NormJob* d_jobs, int njobs, double* out, cudaStream_t st) {
  if (njobs <= 0) return;
  count_launch();
  k_norm<<<njobs, 256, 0, st>>>(d_jobs, out);
}

// ------------------------------------------------------------------ randn
__device__ __forceinline__ uint64_t splitmix(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

__global__ void k_randn(double* dst, int64_t count, uint64_t seed) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t a = splitmix(seed ^ (2 * (uint64_t)i));
    const uint64_t b = splitmix(seed ^ (2 * (uint64_t)i + 1));
    const double u1 = ((a >> 11) + 1) * (1.0 / 9007199254740993.0);
    const double u2 = (b >> 11) * (1.0 / 9007199254740992.0);
    dst[i] = sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
  }
}

__global__ void k_axpby(double a, const double* __restrict__ x, int64_t ldx, double b, double* y, int64_t ldy,
                        int64_t n, int ncols) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * ncols; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % n, j = e / n;
    y[i + j * ldy] = a * x[i + j * ldx] + b * y[i + j * ldy];
  }
}

void launch_axpby(double a, const double* x, int64_t ldx, double b, double* y, int64_t ldy, int64_t n, int ncols,
                  cudaStream_t st) {
  if (n <= 0 || ncols <= 0) return;
  count_launch();
  k_axpby<<<592, 256, 0, st>>>(a, x, ldx, b, y, ldy, n, ncols);
}

void launch_randn(double* dst, int64_t count, uint64_t seed, cudaStream_t st) {
  if (count <= 0) return;
  count_launch();
  k_randn<<<1184, 256, 0, st>>>(dst, count, seed);
}

// ------------------------------------------------------------------ matvec
// y += alpha op(G) x over all leaves (one CTA per leaf, FP64 atomics).
// part (factor views of an in-place H-LR / H-Cholesky, SURVEY O10 probes):
//   0 all of G; 1 L (strict lower + unit diagonal); 2 R (upper incl. diagonal);
//   3 L of Cholesky (lower incl. diagonal); 4 its transpose (call with trans=1).
__global__ void __launch_bounds__(256) k_matvec(const LeafDesc* __restrict__ leaves, int trans,
                                                double alpha, const double* __restrict__ x,
                                                int64_t ldx, double* y, int64_t ldy, int ncols,
                                                int part) {
  __shared__ double tmp[4096];  // k x ncols (host guarantees k*ncols <= 4096)
  const LeafDesc L = leaves[blockIdx.x];
  const bool diag = L.row0 == L.col0 && L.m == L.n;
  if (part != 0 && !diag) {
    const bool lower = L.row0 > L.col0;
    if ((part == 2) == lower) return;   // R: upper blocks only; L parts: lower blocks only
  }
  const int orow = trans ? L.col0 : L.row0, vrow = trans ? L.row0 : L.col0;
  const int mo = trans ? L.n : L.m, ko = trans ? L.m : L.n;
  if (L.kind == 2) {
    for (int64_t e = threadIdx.x; e < (int64_t)mo * ncols; e += 256) {
      const int i = (int)(e % mo), j = (int)(e / mo);
      double s = 0.0;
      for (int p = 0; p < ko; p++) {
        // stored entry (r, c) of the leaf
        const int r = trans ? p : i, cc = trans ? i : p;
        double a = L.A[r + (int64_t)cc * L.m];
        if (part != 0 && diag) {
          if (part == 1) a = (r > cc) ? a : (r == cc ? 1.0 : 0.0);
          else if (part == 2) a = (r <= cc) ? a : 0.0;
          else a = (r >= cc) ? a : 0.0;
        }
        s = fma(a, x[vrow + p + (int64_t)j * ldx], s);
      }
      atomicAdd(&y[orow + i + (int64_t)j * ldy], alpha * s);
    }
  } else if (L.k > 0) {
    const double* F1 = trans ? L.B : L.A;
    const int ld1 = trans ? L.n : L.m;
    const double* F2 = trans ? L.A : L.B;
    const int ld2 = trans ? L.m : L.n;
    for (int e = threadIdx.x; e < L.k * ncols; e += 256) {
      const int q = e % L.k, j = e / L.k;
      double s = 0.0;
      for (int p = 0; p < ko; p++) s = fma(F2[p + (int64_t)q * ld2], x[vrow + p + (int64_t)j * ldx], s);
      tmp[e] = s;
    }
    __syncthreads();
    for (int64_t e = threadIdx.x; e < (int64_t)mo * ncols; e += 256) {
      const int i = (int)(e % mo), j = (int)(e / mo);
      double s = 0.0;
      for (int q = 0; q < L.k; q++) s = fma(F1[i + (int64_t)q * ld1], tmp[q + j * L.k], s);
      atomicAdd(&y[orow + i + (int64_t)j * ldy], alpha * s);
    }
  }
}

void launch_matvec_leaves(const LeafDesc* leaves, int nleaves, int trans, double alpha,
                          const double* x, int64_t ldx, double* y, int64_t ldy, int ncols,
                          int part, cudaStream_t st) {
  if (nleaves <= 0) return;
  count_launch();
  k_matvec<<<nleaves, 256, 0, st>>>(leaves, trans, alpha, x, ldx, y, ldy, ncols, part);
}

__global__ void k_scale(double* y, int64_t ldy, int64_t rows, int cols, double beta) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < rows * cols;
       e += (int64_t)gridDim.x * blockDim.x) {
    double* p = y + (e % rows) + (e / rows) * ldy;
    *p = (beta == 0.0) ? 0.0 : beta * *p;
  }
}

void launch_scale(double* y, int64_t ldy, int64_t rows, int cols, double beta, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return;
  count_launch();
  k_scale<<<592, 256, 0, st>>>(y, ldy, rows, cols, beta);
}

}  // namespace hm
