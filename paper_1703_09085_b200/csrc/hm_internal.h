// libhm internals: context, trees, matrices, device arena, profiling.
#pragma once
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <memory>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/hm.h"
#include "kernels.h"

namespace hm {

struct Error : std::runtime_error {
  hm_status code;
  Error(hm_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define HM_CUDA(call)                                                                 \
  do {                                                                                \
    cudaError_t e_ = (call);                                                          \
    if (e_ != cudaSuccess)                                                            \
      throw ::hm::Error(HM_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

bool debug_sync();   // HM_DEBUG_SYNC=1: synchronize and check after every launch

#define HM_CHECK_LAUNCH()                                                                      \
  do {                                                                                         \
    HM_CUDA(cudaGetLastError());                                                               \
    if (::hm::debug_sync()) {                                                                  \
      cudaError_t e2_ = cudaDeviceSynchronize();                                               \
      if (e2_ != cudaSuccess)                                                                  \
        throw ::hm::Error(HM_ECUDA, std::string(__FILE__) + ":" + std::to_string(__LINE__) + \
                                        ": " + cudaGetErrorString(e2_));                       \
    }                                                                                          \
  } while (0)

enum ProfClass {
  PC_QR = 0, PC_GEMM_M, PC_SVD, PC_APPLYQ, PC_COPY, PC_EVAL, PC_DENSE, PC_MEMSET,
  PC_GEN, PC_BUILD_GEMM, PC_NORM, PC_MATVEC, PC_SVD_B0, PC_SVD_B1, PC_SVD_B2, PC_SVD_B3, PC_QR_SMALL, PC_QR_B0, PC_QR_B1, PC_QR_B2, PC_QR_B3, PC_PREQR, PC_TRSM, PC_LEAF, PC_FUSED, PC_TSQR, PC_COUNT
};

struct Ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  hm_allocator alloc{};
  bool has_alloc = false;
  cudaMemPool_t pool = nullptr;   // private stream-ordered pool (no allocator hook)
  std::set<void*> live;            // hm_mat handles owned by this context
  // standalone batched-flush capture (hm_flush_capture / hm_flush_replay):
  // per level of the next hm_addmul the TRUNC batch's shapes and ranks, and for
  // the levels in cap_mask a device copy of the stacked factors (consumed by
  // the TRUNC, so replays restore them from this copy)
  struct CapLevel {
    std::vector<int> m, n, l, k;
    std::vector<size_t> aoff, boff;   // doubles, relative to data
    double* data = nullptr;
    size_t ndoubles = 0;
  };
  bool cap_on = false;
  uint64_t cap_mask = 0;
  std::vector<CapLevel> cap;
  void cap_free();
  std::string err;
  hm_stats_t last{};
  // profiling
  bool prof = false;
  struct Pending { int cls; cudaEvent_t a, b; double flops, bytes; std::string note; };
  // HM_PROF_LOG=<file>: one line per profiled launch group (class, ms, note)
  std::string note;            // consumed by the next prof_end
  FILE* plog = nullptr;
  cudaEvent_t pbase = nullptr;   // timeline origin of the log (first profiled launch)
  void prof_note(const std::string& s) { if (prof && plog) note = s; }
  std::vector<Pending> pend;
  std::vector<cudaEvent_t> free_events;
  double ms[PC_COUNT] = {0};
  int64_t launches[PC_COUNT] = {0};
  double flops[PC_COUNT] = {0};
  double bytes[PC_COUNT] = {0};

  // pinned staging for job-descriptor uploads: bump allocation, recycled only
  // after the stream has been synchronized (so in-flight copies are complete)
  char* pin = nullptr;
  size_t pin_cap = 0, pin_used = 0;
  // Arena::upload_t: arrays up to this size are read in place.  Off by default
  // (measured on B200: no effect on the H-LR, 9.59 vs 9.60 s at n = 81920 -- the
  // descriptor copies are not on the critical path); HM_ZERO_COPY=1 enables it.
  size_t zc_max = [] { const char* e = std::getenv("HM_ZERO_COPY"); return (e && e[0] == '1') ? (size_t)32 << 10 : (size_t)0; }();
  void* pinned(size_t bytes);
  void pinned_reset() { pin_used = 0; }
  // Rank read-back of small TRUNC batches (the latency-bound factorization
  // steps): the kernels write the ranks straight into mapped pinned host
  // memory, so the host reads them after the stream synchronisation without a
  // blocking cudaMemcpy.  One outstanding batch at a time (reset by the reader);
  // nullptr if the batch is too large (the caller then uses device memory).
  int* rank_host = nullptr;
  size_t rank_cap = 0, rank_used = 0;
  int* rank_alloc(size_t n);
  bool rank_is_host(const int* p) const { return rank_host && p >= rank_host && p < rank_host + rank_cap; }
  // grow-only device workspace for the per-level stacks (one user at a time,
  // stream ordered): avoids re-mapping tens of GB every level
  double* ws = nullptr;
  size_t ws_cap = 0;
  double* stack_ws(size_t ndoubles);
  // Give back the grow-only workspaces (level stacks, LIFO pool, captured
  // flush data) and the private pool's cached memory (hm_trim; also at the
  // start of hm_build, whose temporaries are the largest allocations).
  void trim(bool captures = true);
  // grow-only LIFO pool for arenas in stack mode (factor outputs of one
  // operation); overflow falls back to cudaMallocAsync chunks and the pool is
  // resized to the high-water mark at the next operation start
  char* sp = nullptr;
  size_t sp_cap = 0, sp_top = 0, sp_hwm = 0;
  void sp_prepare();   // call when no stack-mode arena is live
  ~Ctx();

  // every device allocation of the library goes through these two (allocator
  // hook if given, else the private pool)
  void* dmalloc(size_t bytes);
  void dfree(void* p, size_t bytes);
  cudaEvent_t get_event();
  void prof_begin(int cls, cudaEvent_t* a, cudaStream_t st = nullptr);
  void prof_end(int cls, cudaEvent_t a, double flops, double bytes, cudaStream_t st = nullptr);
  // auxiliary streams: independent kernel groups of one TRUNC batch (the fused
  // small stacks, the QR / SVD shared-memory buckets) run side by side.
  // fork(i): aux[i] waits for everything enqueued on `stream` so far;
  // join(i): `stream` waits for aux[i].  HM_STREAMS=0: everything on `stream`.
  static constexpr int kAux = 5;
  cudaStream_t aux[kAux] = {nullptr, nullptr, nullptr, nullptr, nullptr};
  cudaEvent_t ev_fork = nullptr, ev_join[kAux] = {nullptr, nullptr, nullptr, nullptr, nullptr};
  bool multi_stream();
  cudaStream_t fork(int i);
  void join(int i);
  void prof_collect();   // synchronizes pending events
};

// Stream-ordered device arena: bump allocation inside large chunks (few
// cudaMallocAsync calls per level); everything is released by release().
struct Arena {
  Ctx* ctx;
  std::vector<std::pair<void*, size_t>> blocks;
  char* cur = nullptr;
  size_t cur_left = 0;
  size_t chunk_min = (size_t)64 << 20;
  bool stack_mode = false;   // bump-allocate from ctx->sp (LIFO), release to mark
  size_t mark = 0;
  explicit Arena(Ctx* c, bool stack = false) : ctx(c), stack_mode(stack), mark(stack ? c->sp_top : 0) {}
  ~Arena() { release(); }
  void* alloc_bytes(size_t bytes);
  double* alloc(size_t ndoubles) { return static_cast<double*>(alloc_bytes(ndoubles * sizeof(double))); }
  template <class T>
  T* upload(const std::vector<T>& v) {
    if (v.empty()) return nullptr;
    const size_t bytes = v.size() * sizeof(T);
    T* d = static_cast<T*>(alloc_bytes(bytes));
    void* h = ctx->pinned(bytes);
    std::memcpy(h, v.data(), bytes);
    HM_CUDA(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, ctx->stream));
    return d;
  }
  // Transient job descriptors (read once by the kernels enqueued before the
  // owner's next stream synchronisation): small arrays are NOT copied to the
  // device -- the kernels read the pinned, mapped staging memory directly
  // (UVA), which saves one H2D copy (host call + copy-engine latency on the
  // stream) per launch on the latency-bound paths.  HM_ZERO_COPY=0: always copy.
  template <class T>
  T* upload_t(const std::vector<T>& v) {
    if (v.empty()) return nullptr;
    const size_t bytes = v.size() * sizeof(T);
    if (bytes > ctx->zc_max) return upload(v);
    void* h = ctx->pinned(bytes);
    std::memcpy(h, v.data(), bytes);
    return static_cast<T*>(h);
  }
  template <class J>
  const int* tile_map_t(const std::vector<J>& v, int64_t ntiles) {
    if (v.empty() || ntiles <= 0) return nullptr;
    if ((size_t)ntiles * sizeof(int) > ctx->zc_max) return tile_map(v, ntiles);
    std::vector<int> m((size_t)ntiles);
    for (size_t j = 0; j < v.size(); j++) {
      const int64_t t1 = j + 1 < v.size() ? v[j + 1].tile0 : ntiles;
      for (int64_t t = v[j].tile0; t < t1; t++) m[(size_t)t] = (int)j;
    }
    return upload_t(m);
  }
  // job index of every tile of a tiled launch (jobs carry a prefix-summed
  // tile0), uploaded next to the jobs: one load per CTA instead of a binary
  // search of dependent loads
  template <class J>
  const int* tile_map(const std::vector<J>& v, int64_t ntiles) {
    if (v.empty() || ntiles <= 0) return nullptr;
    std::vector<int> m((size_t)ntiles);
    for (size_t j = 0; j < v.size(); j++) {
      const int64_t t1 = j + 1 < v.size() ? v[j + 1].tile0 : ntiles;
      for (int64_t t = v[j].tile0; t < t1; t++) m[(size_t)t] = (int)j;
    }
    return upload(m);
  }
  void release();
};

struct ProfScope {
  Ctx* c;
  int cls;
  double fl, by;
  cudaEvent_t a = nullptr;
  cudaStream_t st;
  ProfScope(Ctx* c_, int cls_, double fl_ = 0, double by_ = 0, cudaStream_t st_ = nullptr)
      : c(c_), cls(cls_), fl(fl_), by(by_), st(st_) {
    c->prof_begin(cls, &a, st);
  }
  ~ProfScope() { c->prof_end(cls, a, fl, by, st); }
};

// Cluster tree + block tree, breadth-first numbered.
struct Tree {
  int64_t n = 0;
  std::vector<int32_t> cl_start, cl_size, cl_son0, cl_nsons, cl_level;
  std::vector<double> cl_bbox;
  std::vector<int32_t> bl_row, bl_col, bl_kind, bl_son0, bl_nsons, bl_level;
  std::vector<int64_t> perm;
  // derived
  std::vector<int32_t> leaf_order;        // leaf block ids in DFS order
  std::vector<int32_t> bl_lbeg, bl_lend;  // DFS leaf range of every block
  int depth = 0;
  int nclusters() const { return (int)cl_start.size(); }
  int nblocks() const { return (int)bl_row.size(); }
  int son(int b, int i, int j) const {   // block son (t_i, s_j)
    return bl_son0[b] + i * cl_nsons[bl_col[b]] + j;
  }
  void finalize();                        // leaf ranges, depth
  bool same_structure(const Tree& o) const;
};

std::shared_ptr<Tree> build_trees(const double* pts, int64_t n, int leaf_size, double eta);

// H-matrix: leaf payload pointers into owned device allocations.
struct Mat {
  std::shared_ptr<Tree> tree;
  std::vector<int32_t> rank;       // per block
  std::vector<double*> pA, pB;     // adm: A, B ; dense: pA = N
  std::pair<void*, size_t> fpool{nullptr, 0};   // admissible-leaf factors
  std::pair<void*, size_t> dpool{nullptr, 0};   // inadmissible-leaf entries
  // export staging
  std::vector<int32_t> ex_rank;
  std::vector<int64_t> ex_off;
  std::unique_ptr<double[]> ex_factors, ex_dense;   // export buffers (uninitialised, owned)
  // geometry kept by hm_build (for diagnostics)
  int kernel = 0;
  void free_all(Ctx* c);
};

std::vector<LeafDesc> leaf_table(const Mat& m);

// Batched TRUNC_eps: independent stacks -> (U_k, V_k S_k), ranks on device.
struct TruncReq {
  int m, n, l;
  double* A;      // m x l (ld m), consumed
  double* B;      // n x l (ld n), consumed
  double* Aout;   // m x kcap (ld m)
  double* Bout;   // n x kcap (ld n)
  int* d_rank;
  double* d_sigma;
};
int trunc_kcap(int m, int n, int l);
void trunc_batched(Ctx* c, Arena& ar, const std::vector<TruncReq>& reqs, double eps);

// SURVEY §8(d) convention flops/bytes of one truncation.
double trunc_flops(double m, double n, double l, double k);
double trunc_bytes(double m, double n, double l, double k);

void addmul(Ctx* c, double alpha, Mat* X, Mat* Y, Mat* Z, double eps);
void addmul_std(Ctx* c, double alpha, Mat* X, Mat* Y, Mat* Z, double eps);
void solve_thin(Ctx* c, Mat* F, int part, double* x, int64_t ldx, int ncols);
double precond_error(Ctx* c, Mat* G0, Mat* F, int kind, int iters, uint64_t seed);
void invert_matrix(Ctx* c, Mat* G, double eps, double* min_pivot);
void flush_replay(Ctx* c, int level, double eps, int reps, double* ms_out, int64_t* rank_sum);
void eval_batched_test(Ctx* c, Mat* H, int njobs, const int* blk, const int* trans, const double* coef,
                       const double* const* V, const int* ldv, double* const* out, const int* ldo, const int* w,
                       double split_thr);
void factorize(Ctx* c, Mat* G, double eps, bool chol, double shift, double* min_pivot);
Mat* build_matrix(Ctx* c, const double* pts, const double* area, const double* nrm, int64_t n, int kernel,
                  int leaf_size, double eta, double eps, int64_t* perm_out);
void matvec(Ctx* c, Mat* G, int op, double alpha, const double* x, int64_t ldx, double beta,
            double* y, int64_t ldy, int ncols);

}  // namespace hm
