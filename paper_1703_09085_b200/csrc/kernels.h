// Batched FP64 kernels for sm_100a (libhm internal).  Every launcher takes a
// device array of job descriptors and enqueues ONE kernel on `st`.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace hm {

// C = alpha * op(A) * op(B) + beta * C   (column-major, per-job shapes)
// mask bit 1: the STORED operand is upper triangular (entries below the
// diagonal of the stored matrix read as 0) -- used for R factors that share
// storage with Householder vectors.
struct GemmJob {
  const double* A;
  const double* B;
  double* C;
  int m, n, k;
  int lda, ldb, ldc;
  int transA, transB;
  int maskA, maskB;
  double alpha, beta;
  int64_t tile0;       // first 64x64 tile id of this job (prefix sum)
  const int* kdyn;     // optional: if non-null, k = *kdyn (device-known width)
  const int* ndyn;     // optional: if non-null, n = *ndyn
};

// In-place Householder QR of a tall panel A (m x n, m > n, lda):
// R in the upper triangle, reflector v_j below the diagonal (v_j[0] = 1
// implicit), tau[j].  LAPACK dgeqr2 convention.
struct QrJob {
  double* A;
  int m, n, lda;
  double* tau;
  double* T;           // optional (k_qr_blocked with 16-column panels, see qr_has_T):
                       // compact-WY T factor of panel p at T + 256 p (16 x 16, upper)
};
// True iff the QR of an m x n panel runs k_qr_blocked with 16-column panels
// (hm_trunc's routing) and can therefore emit the T factors for k_applyq.
inline bool qr_has_T(int m, int n) { return (int64_t)m * n > 4 * 1024 && m <= 1536; }

// X <- Q X with Q = H_0 H_1 ... H_{r-1} from a QrJob (X: m x c, ldx); c is the
// host-side column bound, the actual count is read from *cdyn (device) when
// cdyn != nullptr.  T: the QR's compact-WY panel factors (nullable).
struct ApplyQJob {
  const double* V;     // reflectors (m x r, ldv)
  const double* tau;
  int m, r, ldv;
  double* X;
  int ldx, c;
  const int* cdyn;
  const double* T;
};

// SVD of M (p x q, ldm; QRCP + one-sided Jacobi, svd.cu) + eps rank rule +
// factor output with M ~= Aout Bout^T, *rank = k:
//   the factor on the SHORT side of M (Bout if p >= q, else Aout) is
//   orthonormal (right / left singular vectors), the other one carries the
//   singular values; rows beyond p (Aout) / q (Bout) up to ma / nb are zeroed.
//   sigma[0:min(p,q)] (descending) if sigma != nullptr.
struct SvdJob {
  const double* M;
  int p, q, ldm;
  double* Aout;
  int lda, ma;
  double* Bout;
  int ldb, nb;
  int* rank;
  double* sigma;
  double* work;        // global work (svd_smem_need doubles) when it does not fit smem
  int* nsweep;         // optional: number of Jacobi sweeps used (diagnostics)
  int maskM;           // M is upper triangular (entries below the diagonal read as 0)
};
int svd_smem_need(int p, int q);   // doubles of workspace of one SvdJob

// Fused TRUNC_eps of a small stack (everything in shared memory); one of the
// two output factors is orthonormal (see SvdJob).
struct TruncSmallJob {
  const double* A;     // m x l (ld m)
  const double* B;     // n x l (ld n)
  int m, n, l;
  double* Aout;        // m x k (ld m)
  double* Bout;        // n x k (ld n)
  int* rank;
  double* sigma;
};
int trunc_small_need(int m, int n, int l);   // doubles of shared memory
void launch_trunc_small(const TruncSmallJob* d_jobs, int njobs, double eps, int cap, cudaStream_t st);

// dst[0:rows, 0:cols] (+)= coef * op(src); identity: dst[d,d] = coef.
struct CopyJob {
  double* dst;
  const double* src;
  int ldd, lds, rows, cols;
  int trans, identity, accumulate;
  double coef;
  int64_t tile0;
  int upper;           // copy only the upper triangle of op(src), zeros below
};

// A leaf of an H-matrix in DFS order (for addeval / addevaltrans).
struct LeafDesc {
  int kind;            // 1 admissible, 2 dense
  int row0, col0;      // absolute starts (tree order)
  int m, n, k;
  const double* A;     // adm: m x k ; dense: N (m x n)
  const double* B;     // adm: n x k
};

struct LeafPatch {
  int pos;             // index into a device leaf table
  LeafDesc leaf;
};
void launch_patch_leaves(LeafDesc* table, const LeafPatch* d_patch, int n, cudaStream_t st);

constexpr int kEvalRanges = 8;
// out += coef * H|_{t x s} V   (trans=0; out rows = #t, V rows = #s) or
// out += coef * H|_{t x s}^T V (trans=1; out rows = #s, V rows = #t),
// summed over the leaves [leaf_begin, leaf_end) of block (t,s)  (Fig. 1).
// V(p, j) = vtrans ? V[j + p*ldv] : V[p + j*ldv]; videntity: V = I.
struct EvalJob {
  const LeafDesc* leaves;
  int leaf_begin, leaf_end;
  int trans;
  int t0, s0;
  double coef;
  double* out;
  int ldo, w;
  const double* V;
  int ldv, vtrans, videntity;
  // k_eval2: nrng = 0 visits [leaf_begin, leaf_end) (the whole block); else the
  // leaf ranges rng[0:nrng] = a row group of the block (every range writes
  // output rows no other job of the batch writes), so one large block can be
  // spread over several CTAs without atomics.
  int nrng;
  const int2* rng;
  // chain (identity pre-summing): after this job the same CTA runs *next, which
  // accumulates into the same output columns (sequential: no atomics)
  const EvalJob* next;
};

// Triangular solve through the H-structure on a thin panel (one CTA per job).
// kind 0: V[r0:r0+m] <- T^{-1} V[r0:r0+m], T lower: T(i,j) = trans ? P[j+i ld] : P[i+j ld],
//         unit diagonal if unit;
// kind 1: V -= op(H) V over the leaves [lb, le) (eval semantics, t0 = s0 = panel0).
struct TrsmStep {
  int kind;
  int r0, m;
  const double* P;
  int ld, trans, unit;
  int lb, le;
  int rev;             // kind 0: T is UPPER triangular (backward substitution, run as a forward
                       // substitution in reversed row order)
};
// y = a x + b y (n x ncols panels)
void launch_axpby(double a, const double* x, int64_t ldx, double b, double* y, int64_t ldy, int64_t n, int ncols,
                  cudaStream_t st);
struct TrsmJob {
  double* V;
  int ldv, ncols;
  int panel0;          // absolute start (tree order) of the panel's first row
  int step0, step1;
};

// In-place dense LU (no pivoting, unit L) or Cholesky of a diagonal leaf
// (whole leaf in shared memory: m <= kMaxLeafFactor).
constexpr int kMaxLeafFactor = 160;
struct LeafFactorJob {
  double* N;
  int m, ld;
  int cluster;
};

// Kernel-matrix generation: dst[i,j] = G(perm[r0+i], perm[c0+j]).
struct GenJob {
  double* dst;
  int ld, m, n, r0, c0;
  int64_t tile0;
};

// Frobenius norm squared of a column-major panel -> out[job].
struct NormJob {
  const double* A;
  int m, n, lda;
  const int* ndyn;
};

void launch_gemm(const GemmJob* d_jobs, int njobs, int64_t ntiles, cudaStream_t st);
void launch_gemm_mapped(const GemmJob* d_jobs, int njobs, const int* d_tmap, int64_t ntiles, cudaStream_t st);
void launch_qr(const QrJob* d_jobs, int njobs, int cap, cudaStream_t st);
void launch_qr_blocked(const QrJob* d_jobs, int njobs, int cap, cudaStream_t st);
// Stepped variant (panel kernel + multi-CTA DMMA trailing update per 16
// columns); jobs sorted by n descending, ncols = host copy of their n; every
// job has a T buffer and m <= 1536 (max_m = the largest m).
void launch_qr_stepped(const QrJob* d_jobs, const int* ncols, int njobs, int max_m, cudaStream_t st);   // rows <= 24576
// Register-panel blocked QR (qr_reg.cu): every job n < m <= 768 (max_m = the
// largest m); writes the compact-WY T factors when QrJob::T != nullptr.
void launch_qr_reg(const QrJob* d_jobs, int njobs, int max_m, cudaStream_t st);
// Panel-wise apply-Q on the tensor pipe (qr_reg.cu): every job T != nullptr, m <= 1536.
void launch_applyq_dmma(const ApplyQJob* d_jobs, int njobs, int cmax, int max_m, cudaStream_t st);
void launch_applyq(const ApplyQJob* d_jobs, int njobs, int cmax, cudaStream_t st);
void launch_svd(const SvdJob* d_jobs, int njobs, double eps, int cap, cudaStream_t st);
// k_svd spill mode (C in shared memory for the QRCP, parked in SvdJob::work, X in its place)
bool svd_spill_fits(int p, int q);
void launch_svd_spill(const SvdJob* d_jobs, int njobs, double eps, cudaStream_t st);
void launch_copy(const CopyJob* d_jobs, int njobs, int64_t ntiles, cudaStream_t st);
void launch_copy_mapped(const CopyJob* d_jobs, int njobs, const int* d_tmap, int64_t ntiles, cudaStream_t st);
void launch_eval2(const EvalJob* d_jobs, int njobs, cudaStream_t st);   // eval.cu (shared-memory tiles)
void launch_trsm2(const TrsmJob* d_jobs, int njobs, const TrsmStep* d_steps, const LeafDesc* leaves,
                  cudaStream_t st);   // eval.cu (shared-memory substitution + eval tiles)
void launch_leaf_factor(const LeafFactorJob* d_jobs, int njobs, int chol, int* fail, double* minpiv,
                        int maxm, cudaStream_t st);
void launch_leaf_inverse(const LeafFactorJob* d_jobs, int njobs, int* fail, double* minpiv, int maxm,
                         cudaStream_t st);
void launch_zero_ranges(double* const* d_ptr, const int64_t* d_cnt, int n, cudaStream_t st);
void launch_gen(const GenJob* d_jobs, int njobs, int64_t ntiles, const double* x,
                const double* w, const double* nrm, const int64_t* perm, int kernel, cudaStream_t st);
void launch_norm(const NormJob* d_jobs, int njobs, double* out, cudaStream_t st);
void launch_randn(double* dst, int64_t count, uint64_t seed, cudaStream_t st);
void launch_matvec_leaves(const LeafDesc* leaves, int nleaves, int trans, double alpha,
                          const double* x, int64_t ldx, double* y, int64_t ldy, int ncols,
                          int part, cudaStream_t st);
void launch_scale(double* y, int64_t ldy, int64_t rows, int cols, double beta, cudaStream_t st);

// cudaFuncAttributeMaxDynamicSharedMemorySize for `func` on the CURRENT device,
// set once per (function, device) under a mutex; throws (HM_ECUDA) on failure.
void ensure_smem_attr(const void* func, int bytes);

int64_t launch_count();     // process-wide number of kernel launches
void count_launch();        // called by every launcher
int svd_smem_capacity();   // doubles available for the smem Jacobi path
int qr_smem_capacity();

}  // namespace hm
