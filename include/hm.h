/*
 * hm.h -- C-ABI of libhm: B200-native (sm_100a, FP64) accumulated-update
 * H-matrix arithmetic after S. Boerm, "Hierarchical matrix arithmetic with
 * accumulated updates", arXiv 1703.09085 (cited as P:L<line> of PAPER.md).
 *
 * Plain C99.  No C++ or torch types cross this boundary: only opaque
 * handles, plain host/device pointers, sizes and status codes.  No
 * exception crosses the ABI; every call returns hm_status.
 *
 * Data conventions (all calls)
 *   - FP64 everywhere; dense panels and factors column-major with leading
 *     dimension = number of rows.
 *   - Vectors/panels exchanged with hm_matvec_thin are in TREE order
 *     (cluster index sets are contiguous); hm_build returns the permutation
 *     tree position -> original point index.
 *   - Device pointers passed in are BORROWED (caller-owned, e.g. a torch
 *     tensor's data_ptr()) and must stay valid until the stream passes the
 *     call.  Every hm_mat and all internal pools are OWNED by the context:
 *     an hm_mat is released by hm_free, and hm_ctx_destroy releases every
 *     hm_mat still alive in the context (their handles become invalid).
 *     All device memory of the library comes from the allocator hook, or,
 *     without one, from a PRIVATE stream-ordered pool of the context (the
 *     device's default pool is not modified); hm_ctx_destroy returns it.
 *   - Truncation (TRUNC_eps): the rank k is the smallest k with
 *     sum_{i>k} s_i^2 <= eps^2 sum_i s_i^2 (relative Frobenius, local to the
 *     block, no rank cap; k = 0 for a zero matrix).  Of the two returned
 *     factors exactly ONE is orthonormal: the one on the SHORT side of the
 *     matrix the SVD runs on (see hm_test_trunc_batched); the other carries
 *     the singular values.  Only the represented matrix A B^T is specified.
 *   - Calls are stream-ordered on the context's stream.  Calls that return
 *     host data (hm_build, hm_import, hm_export, hm_stats, hm_addmul's rank
 *     bookkeeping) synchronize the stream.
 *   - Errors: argument / shape errors return HM_EINVAL before any work;
 *     X or Y aliasing Z returns HM_ESTRUCT (use hm_clone for X = Y = Z);
 *     CUDA faults return HM_ECUDA; a message is kept in hm_last_error().
 *   - There is no CPU fallback: every arithmetic step of hm_addmul,
 *     hm_matvec_thin and hm_build runs in this library's sm_100a kernels.
 */
#ifndef HM_H_
#define HM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct hm_ctx_s* hm_ctx;
typedef struct hm_mat_s* hm_mat;

typedef enum {
  HM_OK = 0,
  HM_EINVAL = -1,        /* bad argument / shape */
  HM_ENOMEM = -2,        /* device or host allocation failed */
  HM_ECUDA = -3,         /* CUDA runtime error (incl. asynchronous faults) */
  HM_EPIVOT = -4,        /* numerical breakdown of a leaf factorization */
  HM_ESTRUCT = -5,       /* incompatible trees or aliasing of X/Y with Z */
  HM_EUNSUPPORTED = -6   /* operation not available in this build */
} hm_status;

/* G (single layer), (G + G^T)/2, K + I/2 (double layer) */
enum { HM_KERNEL_SLP = 0, HM_KERNEL_SLP_SYM = 1, HM_KERNEL_DLP = 2 };
/* hm_matvec_thin operators: G, G^T, and (after hm_lr / hm_chol, in place)
 * the unit lower factor L, the upper factor R, the Cholesky factor L and L^T. */
enum { HM_OP_G = 0, HM_OP_GT = 1, HM_OP_L = 2, HM_OP_R = 3, HM_OP_LC = 4, HM_OP_LCT = 5 };

/* Block kinds (Def 2.2 / Def 2.4). */
enum { HM_BLOCK_SUB = 0, HM_BLOCK_ADM = 1, HM_BLOCK_DENSE = 2 };

/*
 * Flat host description of an H-matrix (cluster tree, block tree, leaf
 * payloads).  Trees are breadth-first numbered: the sons of a node are
 * consecutive (son0 .. son0+nsons-1), block sons row-major over
 * sons(t) x sons(s) (Def 2.2).  Payloads:
 *   admissible leaf b (rank k, m = #t, n = #s): A_b = factors[off .. off+m*k)
 *     (m x k), B_b = factors[off+m*k .. off+(m+n)*k) (n x k); G|_b = A_b B_b^T
 *   dense leaf b: N_b = dense[off .. off+m*n) (m x n)
 * Ownership: for hm_import the arrays are caller-owned and read during the
 * call only; for hm_export they are owned by the hm_mat and valid until the
 * next hm_export on it or hm_free.
 */
typedef struct {
  int64_t n;
  int32_t nclusters;
  const int32_t* cl_start;
  const int32_t* cl_size;
  const int32_t* cl_son0;     /* -1 for leaves */
  const int32_t* cl_nsons;
  const int32_t* cl_level;
  const double* cl_bbox;      /* nclusters x 6: lo[3], hi[3] */
  int32_t nblocks;
  const int32_t* bl_row;      /* row cluster id t */
  const int32_t* bl_col;      /* column cluster id s */
  const int32_t* bl_kind;     /* HM_BLOCK_* */
  const int32_t* bl_son0;
  const int32_t* bl_nsons;
  const int32_t* bl_rank;     /* admissible leaves: k; else 0 */
  const int64_t* bl_off;      /* payload offset (doubles) or -1 */
  const double* factors;
  int64_t nfactors;
  const double* dense;
  int64_t ndense;
  const int64_t* perm;        /* tree position -> original index (may be NULL) */
} hm_host_desc;

/* Statistics of a matrix and of the last operation of the context. */
typedef struct {
  int64_t n;
  int32_t nclusters, nblocks, nadm, ndense, depth;
  int32_t max_rank;
  double mean_rank;
  int64_t factor_doubles, dense_doubles;
  /* last hm_addmul */
  int64_t addproduct_calls;   /* = product-tree nodes */
  int64_t evaluated_terms;
  int64_t truncations;        /* T1 + T2 + T3 + merge truncations */
  int64_t trunc_cols;         /* sum of stacked widths l */
  int64_t merges;
  int64_t dense_adds;
  int64_t levels;
  int64_t kernel_launches;    /* process-wide count of libhm kernel launches so far */
  double flops_trunc;         /* SURVEY §8(d) convention flops */
  double flops_eval;
  double flops_dense;
  double bytes_trunc;         /* SURVEY §8(d) convention bytes */
  double bytes_eval;
  double bytes_dense;
  double min_pivot;           /* last hm_lr / hm_chol: min |pivot| of the leaf factorizations */
} hm_stats_t;

/* Per-kernel-class device timing (CUDA events on the context stream,
 * summed over launches since hm_profile_reset). */
#define HM_NPROF 32
typedef struct {
  char name[HM_NPROF][24];
  double ms[HM_NPROF];
  int64_t launches[HM_NPROF];
  double flops[HM_NPROF];     /* convention flops attributed to the class */
  double bytes[HM_NPROF];     /* convention bytes attributed to the class */
  int32_t count;
} hm_prof_t;

/* Device memory hook (stream-ordered: alloc/free are called with the
 * context's stream); NULL -> a private cudaMemPool of the context. */
typedef struct {
  void* (*alloc)(size_t bytes, void* stream, void* user);
  void (*free)(void* ptr, size_t bytes, void* stream, void* user);
  void* user;
} hm_allocator;

/* Context: binds a device and a CUDA stream (cudaStream_t passed as void*;
 * NULL = the legacy default stream).  One context per host thread. */
hm_status hm_ctx_create(int device, void* cuda_stream, const hm_allocator* alloc, hm_ctx* out);
hm_status hm_ctx_destroy(hm_ctx ctx);
const char* hm_last_error(hm_ctx ctx);
hm_status hm_sync(hm_ctx ctx);
/* Synchronises the stream and gives back the context's grow-only workspaces
 * (level stacks, LIFO pool, captured flush batches) and the memory its private
 * pool has cached; live hm_mat handles are untouched.  The next operation
 * re-grows what it needs.  hm_build / hm_build_nrm call it and retry once
 * when they run out of device memory. */
hm_status hm_trim(hm_ctx ctx);
const char* hm_version(void);

/*
 * hm_build: H-matrix approximation of the BEM-like kernel matrix of
 * BASELINE.json (G_ij = area_j/(4 pi |x_i - x_j|), G_ii = sqrt(area_i/pi)/2;
 * HM_KERNEL_SLP_SYM: (G+G^T)/2).  Trees: bounding-box bisection (longest
 * axis, midpoint) with leaf size `leaf_size`; admissibility
 * max(diam_t, diam_s) <= eta dist(t,s) (squared form).  Dense leaves hold
 * exact entries; admissible leaves TRUNC_eps(G|_b) (relative Frobenius
 * rule), computed on the device from generated entries by a certified
 * randomized range finder (residual <= 1e-12 ||G|_b||_F) followed by the
 * batched TRUNC kernels.
 *   pts_host: n x 3 row-major, area_host: n (host, read during the call)
 *   perm_host: optional, n entries written (tree position -> original)
 */
hm_status hm_build(hm_ctx ctx, const double* pts_host, const double* area_host, int64_t n,
                   int kernel, int leaf_size, double eta, double eps,
                   hm_mat* out, int64_t* perm_host);
/* hm_build_nrm: as hm_build with unit normals nrm_host (n x 3 row-major,
 * outward, host, read during the call; NULL allowed except for
 * HM_KERNEL_DLP): K_ij = area_j ((x_j - x_i) . n_j) / (4 pi |x_i - x_j|^3),
 * K_ii = 1/2 -- the double-layer matrix plus 1/2 I of PAPER.md P:L1583-1585
 * (sign: DESIGN.md reading R20, K 1 ~ 1/2 on a closed surface). */
hm_status hm_build_nrm(hm_ctx ctx, const double* pts_host, const double* area_host, const double* nrm_host,
                       int64_t n, int kernel, int leaf_size, double eta, double eps, hm_mat* out,
                       int64_t* perm_host);

/* hm_import: upload a flat host description (trees + payloads). */
hm_status hm_import(hm_ctx ctx, const hm_host_desc* d, hm_mat* out);
/* hm_export: download; pointers in *d owned by the matrix (see above). */
hm_status hm_export(hm_ctx ctx, hm_mat m, hm_host_desc* d);

/* hm_export_sizes: payload sizes (doubles) hm_export / hm_export_into produce. */
hm_status hm_export_sizes(hm_ctx ctx, hm_mat m, int64_t* nfactors, int64_t* ndense);

/* hm_export_into: as hm_export, but the factor / dense payloads are copied
 * straight into CALLER-owned host buffers factors_out (nfactors doubles) and
 * dense_out (ndense doubles) -- one bulk D2H per pool, no library-side host
 * copy (pinned buffers give full DMA bandwidth).  d->factors / d->dense are
 * set to those buffers; the other arrays of *d are owned by the matrix as for
 * hm_export.  HM_EINVAL if a buffer is null while its size is non-zero. */
hm_status hm_export_into(hm_ctx ctx, hm_mat m, hm_host_desc* d, double* factors_out, double* dense_out);
hm_status hm_clone(hm_ctx ctx, hm_mat src, hm_mat* out);
hm_status hm_free(hm_ctx ctx, hm_mat m);

/*
 * hm_addmul: Z <- blocktrunc(Z + alpha X Y) with accumulated updates
 * (addproduct Fig. 5, split Fig. 6, flush Fig. 7).  X, Y, Z must
 * share one block tree (e.g. clones); Z must not alias X or Y.  The
 * schedule is the level-batched S2 reading: exact terms are
 * truncated once per accumulator at split (T1) or flush (T2/T3), plus the
 * rkmerge truncations (Fig. 4).  eps: relative Frobenius truncation
 * tolerance per block.  Every level of the block tree is one batch of
 * device work; the host reads back only the per-level rank arrays.
 */
hm_status hm_addmul(hm_ctx ctx, double alpha, hm_mat X, hm_mat Y, hm_mat Z, double eps);

/*
 * hm_addmul_std: the STANDARD (immediate-update) product Z <- Z + alpha X Y of
 * PAPER.md §4 -- the paper's baseline the accumulated product
 * is compared against (Fig. 9): every evaluated elementary
 * product is truncated into each admissible Z leaf below its block at once
 * (rkupdate, Fig. 3), temporaries + rkmerge below admissible leaves
 * (P:L871-875).  Same arguments, trees and errors as hm_addmul; the result
 * differs from hm_addmul's by truncation error only (same exact product).
 * hm_stats reports its truncation count (the paper's point: S0 truncates far
 * more often) and `levels` = number of dependent TRUNC rounds.
 */
hm_status hm_addmul_std(hm_ctx ctx, double alpha, hm_mat X, hm_mat Y, hm_mat Z, double eps);

/* H-LR (unit lower L, upper R, in place) and H-Cholesky (lower L, in place,
 * G + shift*I factored) with accumulated updates. */
hm_status hm_lr(hm_ctx ctx, hm_mat G, double eps);
hm_status hm_chol(hm_ctx ctx, hm_mat G, double eps, double shift);

/*
 * hm_inv: G <- approximate G^{-1} in place, H-matrix inversion with
 * accumulated updates (§6, Fig. 8): block LR steps
 * on the binary cluster tree, every update through addproduct / split /
 * flush, an auxiliary H-matrix for H12 / H21 (allocated and
 * released inside the call), dense leaf inverses by Gauss-Jordan without
 * pivoting (the paper assumes invertible principal submatrices,
 * P:L1357-1360).  Reading R21: Fig. 8's last addproduct goes to
 * the (t1,t1) accumulator it is flushed from.  HM_EPIVOT on a singular leaf
 * pivot; hm_stats: truncations etc. of the call, min_pivot.  Synchronizes.
 */
hm_status hm_inv(hm_ctx ctx, hm_mat G, double eps);

/*
 * hm_solve_thin: X <- op(F)^{-1} X in place, F = an hm_lr / hm_chol result,
 * X: n x ncols device panel in tree order (ld ldx >= n).  op:
 *   HM_SOLVE_L (unit lower L), HM_SOLVE_R (upper R), HM_SOLVE_LT (L^T),
 *   HM_SOLVE_RT (R^T), HM_SOLVE_LC (Cholesky L), HM_SOLVE_LCT (L^T).
 * Block substitution through the cluster tree (dense leaf substitutions +
 * Fig. 1 addeval updates); (L R)^{-1} x = two calls (L then R).  The
 * preconditioner of PAPER.md P:L1628-1629.  Synchronizes.
 */
enum { HM_SOLVE_L = 0, HM_SOLVE_R = 1, HM_SOLVE_LT = 2, HM_SOLVE_RT = 3, HM_SOLVE_LC = 4, HM_SOLVE_LCT = 5 };
hm_status hm_solve_thin(hm_ctx ctx, hm_mat F, int op, double* x_dev, int64_t ldx, int ncols);

/*
 * hm_precond_error: the paper's preconditioner error ||I - F^{-1} G||_2
 * ("estimate the spectral norm ... using a power iteration"),
 * F = L R (kind 0, after hm_lr) or L L^T (kind 1, after hm_chol), G the
 * unfactored matrix (e.g. an hm_clone taken before factorizing), or kind 2:
 * F = the approximate inverse from hm_inv (E = I - F G); `iters`
 * power steps on E^T E from a seeded Gaussian start (device generator,
 * `seed`); *out = ||E v|| of the last step (a lower bound converging to
 * ||E||_2).  All vector work on the device; synchronizes.
 */
hm_status hm_precond_error(hm_ctx ctx, hm_mat G, hm_mat F, int kind, int iters, uint64_t seed, double* out);

/*
 * hm_matvec_thin: Y <- alpha op(G) X + beta Y (Fig. 1 addeval/addevaltrans,
 * P:L300-334) for n x ncols device panels in tree order.
 */
hm_status hm_matvec_thin(hm_ctx ctx, hm_mat G, int op, double alpha, const double* x_dev,
                         int64_t ldx, double beta, double* y_dev, int64_t ldy, int ncols);

hm_status hm_stats(hm_ctx ctx, hm_mat m, hm_stats_t* out);

/* Kernel-class timing with CUDA events (off by default). */
hm_status hm_profile_enable(hm_ctx ctx, int on);
hm_status hm_profile_reset(hm_ctx ctx);
hm_status hm_profile_get(hm_ctx ctx, hm_prof_t* out);

/*
 * Test-only export: batched TRUNC_eps of independent stacks (kernel-level
 * parity).  For job i: A_i (m_i x l_i, ld m_i) at a_dev + a_off[i],
 * B_i (n_i x l_i) at b_dev + b_off[i] (device, CONSUMED: overwritten);
 * results A'_i (m_i x k) at ua_dev + o_off[i] (ld m_i) and B'_i (n_i x k)
 * at ub_dev + p_off[i] (ld n_i), capacity min(m,n,l) columns, with
 * A'_i B'_i^T = the eps-truncated SVD of A_i B_i^T; ranks_host[i] = k,
 * sigma_host (optional) the singular values.  Which factor is orthonormal:
 * the SVD runs on M = R_A R_B^T (or A R_B^T / R_A B^T when only one side is
 * QR'd), stored in its tall orientation; the factor belonging to the short
 * side of M is orthonormal (U_k on the A side if M has fewer rows than
 * columns, V_k on the B side otherwise), the other one is scaled by the
 * singular values (reading R7c).  Offsets are host arrays in doubles.
 */
hm_status hm_test_trunc_batched(hm_ctx ctx, int njobs, const int32_t* m, const int32_t* n,
                                const int32_t* l, double* a_dev, const int64_t* a_off,
                                double* b_dev, const int64_t* b_off, double* ua_dev,
                                const int64_t* o_off, double* ub_dev, const int64_t* p_off,
                                double eps, int32_t* ranks_host, double* sigma_host);

/*
 * Test-only export: batched H x thin-dense products (Fig. 1 addeval /
 * addevaltrans) through the launch path of hm_addmul's A2 step
 * (DFS leaf ranges of the block, row-group splitting of large jobs, one
 * k_eval2 batch).  For job i with block b = blk[i] = (t, s) of H:
 *   trans[i] = 0: out_i += coef[i] * H|_{t x s} V_i   (V_i: #s x w[i], out_i: #t x w[i])
 *   trans[i] = 1: out_i += coef[i] * H|_{t x s}^T V_i (V_i: #t x w[i], out_i: #s x w[i])
 * V_i at v_dev + v_off[i] (ld ldv[i]), out_i at out_dev + o_off[i] (ld
 * ldo[i]), device, column-major; outputs of different jobs must not overlap.
 * split_threshold > 0 forces the row-group split of every job whose cost
 * estimate exceeds it (exercises the split path); <= 0: production rule.
 * Synchronizes.
 */
hm_status hm_test_eval_batched(hm_ctx ctx, hm_mat H, int njobs, const int32_t* blk, const int32_t* trans,
                               const double* coef, double* v_dev, const int64_t* v_off, const int32_t* ldv,
                               double* out_dev, const int64_t* o_off, const int32_t* ldo, const int32_t* w,
                               double split_threshold);

/*
 * Standalone batched flush (BASELINE configs[3]: "also timed
 * as standalone batched flush"): the TRUNC_eps batches of the flush of Fig. 7
 * captured in situ during an hm_addmul and replayed alone.
 *   hm_flush_capture(ctx, mask): the NEXT hm_addmul of the context records,
 *     per block-tree level (batch index 0, 1, ... in execution order), the
 *     shapes (m, n, l) and resulting ranks of its TRUNC batch (T1 reduces and
 *     T2/T3 flushes; rkmerge batches excluded), and for the levels whose bit
 *     is set in `mask` a device copy of the stacked factors (up to tens of GB
 *     per level, owned by the context until hm_flush_capture_free).
 *   hm_flush_capture_info(ctx, level, njobs, m, n, l, k, has_data): level < 0:
 *     *njobs = number of captured levels; else *njobs = batch size and, for
 *     non-NULL host arrays of njobs entries, the shapes and ranks.
 *   hm_flush_replay(ctx, level, eps, reps, ms_out, rank_sum): restores the
 *     captured stacks (not timed) and runs the level's TRUNC batch `reps`
 *     times; *ms_out = mean device time of the TRUNC batch (CUDA events on
 *     the context stream), *rank_sum = sum of the resulting ranks (equal to
 *     the in-situ ranks' sum: same inputs, same kernels).  Synchronizes.
 */
hm_status hm_flush_capture(hm_ctx ctx, uint64_t level_mask);
hm_status hm_flush_capture_info(hm_ctx ctx, int level, int64_t* njobs, int32_t* m, int32_t* n, int32_t* l,
                                int32_t* k, int* has_data);
hm_status hm_flush_replay(hm_ctx ctx, int level, double eps, int reps, double* ms_out, int64_t* rank_sum);
hm_status hm_flush_capture_free(hm_ctx ctx);

#ifdef __cplusplus
}
#endif
#endif /* HM_H_ */
