// hm_addmul: Z <- blocktrunc(Z + alpha X Y) with accumulated updates
// (§4: addproduct Fig. 5, split Fig. 6 P:L1028-1050,
// flush Fig. 7), executed level-synchronously.
//
// Accumulators of one block-tree level are processed together: the host
// expands the pending products of level l into the accumulators of level
// l+1 (integer work only) and emits ONE batch of device work per level:
//   gather (copies of base / Z views, explicit factors, identities),
//   eval   (addeval / addevaltrans over DFS leaf ranges, Fig. 1),
//   TRUNC  (T1 reduce at split, T2 flush into admissible Z leaves, T3 flush
//           into temporary Z~ blocks),
//   dense  (exact N_b += A B^T for inadmissible Z leaves).
// Then the rkmerge truncations (Fig. 4, T4) run bottom-up, one batch per
// level.  The schedule is the S2 reading: each accumulator truncates its
// exact stack once (DESIGN.md §3 R2), so the truncated matrices are the
// oracle's (oracle/product.py S2).
#include <algorithm>
#include <atomic>
#include <thread>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <memory>
#include <numeric>
#include <unordered_map>

#include "hm_internal.h"

namespace hm {
namespace {

enum { ZS = 0, ZA = 1, ZD = 2, ZV = 3 };

struct FP {            // device factor pair; rows relative to clusters starting at t0 / r0
  double* A;
  double* B;
  int lda, ldb;
  int t0, r0;
  int k;
};

// Operands carry the index of the H-matrix they belong to (Planner::mats):
// the product has X, Y, Z; the factorizations one matrix G; the inversion of
// Fig. 8 mixes G and the auxiliary H.  alpha is per product.
struct Term {
  int bx, by, br, w;
  bool xd = false, yd = false;   // X|ts / Y|sr is a dense leaf (identity branches 0 / 2 available)
  int xm = 0, ym = 0;
  double alpha = 1.0;
};
struct Pend { int bx, by; int xm, ym; double alpha; };

struct Node {
  int t, r;
  int zt, zb;
  int zm = 0;                 // index (Planner::mats) of the matrix holding block zb
  int base = -1;
  std::vector<Term> terms;
  std::vector<Pend> pend;
  int red = -1;
  int result = -1;
  int child0 = -1;
  bool force_split = false;   // H-LR/H-Cholesky: split (reduce + expand) even with P = 0
  bool no_expand = false;     // reduce only (T1); the caller expands the sons itself
};

struct Planner {
  Ctx* c;
  Arena persist;        // FP outputs (freed at the end of hm_addmul)
  const Tree& T;
  Mat *X, *Y, *Z;
  std::vector<Mat*> mats;     // distinct matrices; X, Y, Z are mats[xm0], mats[ym0], mats[zm0]
  int xm0 = 0, ym0 = 0, zm0 = 0;
  double alpha, eps;
  std::vector<FP> fps;
  std::vector<std::vector<Node>> levels;
  std::vector<std::vector<int>> zresult;   // [matrix][real adm leaf id] -> FP id
  std::vector<std::pair<int, int>> touched;   // (matrix, block) whose zresult was set
  std::vector<std::vector<LeafDesc>> ltab;      // per matrix: leaves in DFS order
  std::vector<std::vector<double>> lmat, lmn;   // DFS prefix sums (convention counts)
  std::vector<LeafDesc*> dltab;                 // device copies of ltab
  double t_wait = 0;
  int64_t n_sync = 0;
  // stats
  int64_t n_addproduct = 0, n_eval = 0, n_trunc = 0, n_cols = 0, n_merge = 0, n_dense = 0;
  double fl_trunc = 0, by_trunc = 0, fl_eval = 0, by_eval = 0, fl_dense = 0, by_dense = 0;

  // Y as a transpose view of a matrix over the same (symmetric) block tree
  // (H-Cholesky: addproduct(-1, L_21, L_21^T)): block (s,r) of the view is
  // block tmap[(s,r)] = (r,s) of *Y, transposed.
  bool ytrans = false;
  std::vector<int> tmap;
  Arena* fp_arena = nullptr;   // where new_fp allocates (default: persist)
  Arena heap;                  // non-LIFO FP outputs that must outlive a flush's local (stack) arena
  bool fp_heap = false;        // new_fp allocates from heap (T1 results of no_expand nodes)

  Planner(Ctx* c_, const Tree& T_, Mat* X_, Mat* Y_, Mat* Z_, double a, double e)
      : c(c_), persist(c_, true), heap(c_, false), T(T_), X(X_), Y(Y_), Z(Z_), alpha(a), eps(e) {
    xm0 = add_mat(X_);
    ym0 = add_mat(Y_);
    zm0 = add_mat(Z_);
  }
  int add_mat(Mat* m) {
    for (size_t i = 0; i < mats.size(); i++)
      if (mats[i] == m) return (int)i;
    mats.push_back(m);
    return (int)mats.size() - 1;
  }
  int& zres(int m, int b) { return zresult[m][b]; }
  void set_zres(int m, int b, int fp) {
    zresult[m][b] = fp;
    touched.push_back({m, b});
  }

  int csize(int cl) const { return T.cl_size[cl]; }
  int cstart(int cl) const { return T.cl_start[cl]; }
  int yb(int by) const { return ytrans ? tmap[by] : by; }

  // Fig. 5 classification in printed branch order.
  bool classify(int bx, int by, Term& out) const { return classify(bx, by, xm0, ym0, out); }
  bool classify(int bx, int by, int xm, int ym, Term& out) const {
    const int kx = T.bl_kind[bx], ky = T.bl_kind[by];
    const int t = T.bl_row[bx], s = T.bl_col[bx], r = T.bl_col[by];
    const Mat* Xm = mats[xm];
    const Mat* Ym = mats[ym];
    out.bx = bx;
    out.by = by;
    out.xm = xm;
    out.ym = ym;
    out.alpha = alpha;
    out.xd = kx == HM_BLOCK_DENSE;
    out.yd = ky == HM_BLOCK_DENSE;
    if (kx == HM_BLOCK_DENSE) {
      if (csize(t) <= csize(s)) { out.br = 0; out.w = csize(t); }
      else { out.br = 1; out.w = csize(s); }
    } else if (ky == HM_BLOCK_DENSE) {
      if (csize(r) <= csize(s)) { out.br = 2; out.w = csize(r); }
      else { out.br = 3; out.w = csize(s); }
    } else if (kx == HM_BLOCK_ADM) {
      out.br = 4; out.w = Xm->rank[bx];
    } else if (ky == HM_BLOCK_ADM) {
      out.br = 5; out.w = Ym->rank[yb(by)];
    } else {
      return false;
    }
    if (narrow) {
      // Any branch whose leaf condition holds factorizes the SAME exact product
      // alpha X|ts Y|sr; pick the narrowest (reading R7b): the
      // truncated matrix is unchanged, only the stack width shrinks.
      auto cand = [&](int br, int w) {
        if (w < out.w) { out.br = br; out.w = w; }
      };
      if (kx == HM_BLOCK_DENSE) cand(csize(t) <= csize(s) ? 0 : 1, std::min(csize(t), csize(s)));
      if (ky == HM_BLOCK_DENSE) cand(csize(r) <= csize(s) ? 2 : 3, std::min(csize(r), csize(s)));
      if (kx == HM_BLOCK_ADM) cand(4, Xm->rank[bx]);
      if (ky == HM_BLOCK_ADM) cand(5, Ym->rank[yb(by)]);
    }
    return true;
  }
  bool narrow = true;

  void addproduct(Node& nd, int bx, int by) { addproduct(nd, bx, by, xm0, ym0, alpha); }
  void addproduct(Node& nd, int bx, int by, int xm, int ym, double a) {
    n_addproduct++;
    Term tm;
    if (classify(bx, by, xm, ym, tm)) {
      tm.alpha = a;
      nd.terms.push_back(tm);
      n_eval++;
    } else {
      nd.pend.push_back(Pend{bx, by, xm, ym, a});
    }
  }

  FP zview(int zb) const { return zview(zm0, zb); }
  FP zview(int zm, int zb) const {
    const Mat* Zm = mats[zm];
    FP f;
    f.A = Zm->pA[zb];
    f.B = Zm->pB[zb];
    f.lda = csize(T.bl_row[zb]);
    f.ldb = csize(T.bl_col[zb]);
    f.t0 = cstart(T.bl_row[zb]);
    f.r0 = cstart(T.bl_col[zb]);
    f.k = Zm->rank[zb];
    return f;
  }

  int new_fp(int m, int n, int kcap, int t0, int r0) {
    FP f;
    Arena& ar = fp_heap ? heap : (fp_arena ? *fp_arena : persist);
    f.A = ar.alloc((size_t)m * std::max(kcap, 1));
    f.B = ar.alloc((size_t)n * std::max(kcap, 1));
    f.lda = m;
    f.ldb = n;
    f.t0 = t0;
    f.r0 = r0;
    f.k = -1;
    fps.push_back(f);
    return (int)fps.size() - 1;
  }

  // ------------------------------------------------------------ level batch
  struct Stack {
    int node;
    int kind;      // 1 T1, 2 T2/T3, 3 dense
    int m, n, l;
    double *A, *B;
    int out = -1;  // FP id
  };

  void add_copy(std::vector<CopyJob>& cj, int64_t& tiles, double* dst, int ldd, const double* src,
                int lds, int rows, int cols, int trans, int identity, double coef) {
    if (rows <= 0 || cols <= 0) return;
    CopyJob j{};
    j.dst = dst; j.src = src; j.ldd = ldd; j.lds = lds; j.rows = rows; j.cols = cols;
    j.trans = trans; j.identity = identity; j.accumulate = 0; j.coef = coef; j.tile0 = tiles;
    tiles += (int64_t)((rows + 31) / 32) * ((cols + 31) / 32);
    cj.push_back(j);
  }

  // H-side product over the DFS leaves of block blk of X (yside = false) or Y
  // (yside = true); trans: out += coef H|_blk^T V instead of H|_blk V.
  struct EvalMeta { double cost; int blk, mat; };
  // Host-side state of one eval batch under construction.  The level batch of
  // hm_addmul is built by several host threads (run_level_enqueue): each
  // worker points tl_emit at its own EmitState; everything else uses `em0`.
  struct EmitState {
    std::vector<EvalMeta> emeta;   // host-side companions of the batch's EvalJobs
    std::vector<int2> erng;        // leaf-range table of split jobs (uploaded with the jobs)
    std::vector<EvalJob> etail;    // chained continuation jobs (identity groups)
    double fl = 0, by = 0;         // convention work emitted by a worker (folded in by the owner)
  };
  EmitState em0;
  static EmitState*& tl_emit() {
    static thread_local EmitState* p = nullptr;
    return p;
  }
  EmitState& em() { return tl_emit() ? *tl_emit() : em0; }
  double split_thr = -1;         // > 0: fixed split threshold (hm_test_eval_batched)

  // H-side product over the DFS leaves of block blk of matrix mats[mi]
  void add_eval(std::vector<EvalJob>& ej, int mi, int blk, int trans, double coef, double* out,
                int ldo, int w, const double* V, int ldv, int vtrans, int videntity) {
    if (w <= 0) return;
    EvalJob e{};
    e.leaves = dltab[mi];
    e.leaf_begin = T.bl_lbeg[blk];
    e.leaf_end = T.bl_lend[blk];
    e.trans = trans;
    e.t0 = cstart(T.bl_row[blk]);
    e.s0 = cstart(T.bl_col[blk]);
    e.coef = coef;
    e.out = out;
    e.ldo = ldo;
    e.w = w;
    e.V = V;
    e.ldv = ldv;
    e.vtrans = vtrans;
    e.videntity = videntity;
    // convention work from DFS prefix sums over the leaf table (O(1) per term):
    // dense leaf 2 m'n' w flops, low-rank leaf 2 k'(m'+n') w; bytes = payload + panels
    const std::vector<double>& pm = lmat[mi];
    const std::vector<double>& pn = lmn[mi];
    const double smat = pm[e.leaf_end] - pm[e.leaf_begin];
    const double smn = pn[e.leaf_end] - pn[e.leaf_begin];
    double fl = videntity ? 0.0 : 2.0 * w * smat;   // expansion: a copy, not arithmetic
    const double by = 8.0 * (smat + smn * w);
    if (tl_emit()) { tl_emit()->fl += fl; tl_emit()->by += by; }
    else { fl_eval += fl; by_eval += by; }
    e.nrng = 0;
    e.rng = nullptr;
    ej.push_back(e);
    em().emeta.push_back(EvalMeta{by + fl, blk, mi});
  }

  // Load balance of one eval batch: a job whose cost exceeds thr is cut into
  // row groups of its block -- the output-row cluster (row cluster for
  // trans = 0, column cluster for trans = 1) is descended while every block of
  // the group is subdivided; each group keeps the DFS ranges of its sub-blocks
  // (at most kEvalRanges) and writes only its own output rows.  The sums per
  // output entry run over the same leaves in the same order, so the result is
  // bit-identical to the unsplit job.
  void split_evals(std::vector<EvalJob>& ej) {
    std::vector<EvalMeta>& emeta = em().emeta;
    std::vector<int2>& erng = em().erng;
    erng.clear();
    double total = 0;
    for (auto& m : emeta) total += m.cost;
    static const double div = [] { const char* e = std::getenv("HM_EVAL_SPLIT"); return e ? std::atof(e) : 1184.0; }();
    if (div <= 0) return;
    const double thr = split_thr > 0 ? split_thr : std::max(total / div, 2e5);
    std::vector<EvalJob> out;
    std::vector<EvalMeta> mout;
    out.reserve(ej.size());
    mout.reserve(ej.size());
    for (size_t ji = 0; ji < ej.size(); ji++) {
      const EvalJob& e = ej[ji];
      const EvalMeta& em = emeta[ji];
      if (em.cost <= thr || e.next) { out.push_back(e); mout.push_back(em); continue; }
      const std::vector<double>& pm = lmat[em.mat];
      const std::vector<double>& pn = lmn[em.mat];
      auto bcost = [&](int b) {
        const double smat = pm[T.bl_lend[b]] - pm[T.bl_lbeg[b]], smn = pn[T.bl_lend[b]] - pn[T.bl_lbeg[b]];
        return 8.0 * (smat + smn * e.w) + (e.videntity ? 0.0 : 2.0 * e.w * smat);
      };
      struct G { std::vector<int> blocks; double cost; };
      std::vector<G> groups{G{{em.blk}, em.cost}};
      for (int it = 0; it < 3; it++) {
        std::vector<G> nx;
        bool any = false;
        for (G& g : groups) {
          bool ok = g.cost > thr;
          int nsplit = 0;
          for (int b : g.blocks) {
            if (T.bl_kind[b] != HM_BLOCK_SUB) { ok = false; break; }
            nsplit = T.cl_nsons[e.trans ? T.bl_col[b] : T.bl_row[b]];
          }
          const int other = ok ? T.cl_nsons[e.trans ? T.bl_row[g.blocks[0]] : T.bl_col[g.blocks[0]]] : 0;
          if (!ok || (int)g.blocks.size() * other > kEvalRanges) { nx.push_back(std::move(g)); continue; }
          any = true;
          for (int i = 0; i < nsplit; i++) {
            G h{{}, 0.0};
            for (int b : g.blocks) {
              const int no = T.cl_nsons[e.trans ? T.bl_row[b] : T.bl_col[b]];
              for (int j = 0; j < no; j++) {
                const int sb = e.trans ? T.son(b, j, i) : T.son(b, i, j);
                h.blocks.push_back(sb);
                h.cost += bcost(sb);
              }
            }
            nx.push_back(std::move(h));
          }
        }
        groups.swap(nx);
        if (!any) break;
      }
      for (G& g : groups) {
        EvalJob s = e;
        // sub-blocks in DFS order; adjacent ranges merged; the range table
        // offset is stored in rng until the table is uploaded
        std::sort(g.blocks.begin(), g.blocks.end(), [&](int a, int b) { return T.bl_lbeg[a] < T.bl_lbeg[b]; });
        const size_t r0 = erng.size();
        for (int b : g.blocks) {
          if (T.bl_lbeg[b] == T.bl_lend[b]) continue;
          if (erng.size() > r0 && erng.back().y == T.bl_lbeg[b]) erng.back().y = T.bl_lend[b];
          else erng.push_back(make_int2(T.bl_lbeg[b], T.bl_lend[b]));
        }
        s.nrng = (int)(erng.size() - r0);
        s.rng = reinterpret_cast<const int2*>(static_cast<intptr_t>(r0));
        if (s.nrng > 0) { out.push_back(s); mout.push_back(EvalMeta{g.cost, em.blk, em.mat}); }
      }
    }
    ej.swap(out);
    emeta.swap(mout);
  }

  // Split (load balance) and sort largest-first: host work only, on the active
  // EmitState (a worker thread's or em0).  The range-table offsets and chain
  // links of the sorted jobs stay relative until submit_evals.
  std::vector<EvalJob> prepare_evals(std::vector<EvalJob>& ej) {
    std::vector<EvalJob> sorted;
    if (ej.empty()) return sorted;
    split_evals(ej);
    const std::vector<EvalMeta>& emeta = em().emeta;
    std::vector<int> order(ej.size());
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return emeta[a].cost > emeta[b].cost; });
    sorted.resize(ej.size());
    for (size_t i = 0; i < order.size(); i++) sorted[i] = ej[order[i]];
    em().emeta.clear();
    ej.clear();
    return sorted;
  }

  // Upload one prepared batch (jobs, range table, chained jobs of state E) and launch k_eval2.
  // aux >= 0: the kernel runs on auxiliary stream `aux` (forked after the uploads;
  // the caller joins it), so consecutive batches overlap their tails
  void submit_evals(std::vector<EvalJob>& sorted, EmitState& E, Arena& scratch, double fl, double by, int aux = -1) {
    if (sorted.empty()) return;
    const int2* drng = E.erng.empty() ? nullptr : scratch.upload_t(E.erng);
    EvalJob* dtail = nullptr;
    if (!E.etail.empty()) {
      dtail = static_cast<EvalJob*>(scratch.alloc_bytes(E.etail.size() * sizeof(EvalJob)));
      for (auto& t : E.etail)
        if (t.next) t.next = dtail + (reinterpret_cast<intptr_t>(t.next) - 1);
      void* h = c->pinned(E.etail.size() * sizeof(EvalJob));
      std::memcpy(h, E.etail.data(), E.etail.size() * sizeof(EvalJob));
      HM_CUDA(cudaMemcpyAsync(dtail, h, E.etail.size() * sizeof(EvalJob), cudaMemcpyHostToDevice, c->stream));
    }
    for (EvalJob& j : sorted) {
      if (j.nrng > 0) j.rng = drng + reinterpret_cast<intptr_t>(j.rng);
      if (j.next) j.next = dtail + (reinterpret_cast<intptr_t>(j.next) - 1);
    }
    E.erng.clear();
    E.etail.clear();
    const EvalJob* dj = scratch.upload_t(sorted);
    cudaStream_t st = aux >= 0 ? c->fork(aux) : c->stream;
    ProfScope ps(c, PC_EVAL, fl, by, st);
    launch_eval2(dj, (int)sorted.size(), st);
    HM_CHECK_LAUNCH();
    sorted.clear();
  }

  void launch_evals(std::vector<EvalJob>& ej, Arena& scratch, double fl, double by) {
    if (ej.empty()) return;
    std::vector<EvalJob> sorted = prepare_evals(ej);
    submit_evals(sorted, em(), scratch, fl, by);
  }

  // Emit the A2 realisation of one evaluated term into stack columns [col, col+w).
  void emit_term(const Term& tm, double* SA, int m, double* SB, int n, int col,
                 std::vector<CopyJob>& cj, int64_t& ctiles, std::vector<EvalJob>& ej) {
    const int bx = tm.bx, by = tm.by, w = tm.w;
    const int t = T.bl_row[bx], s = T.bl_col[bx], r = T.bl_col[by];
    const int nt = csize(t), ns = csize(s), nr = csize(r);
    double* a = SA + (size_t)col * m;
    double* b = SB + (size_t)col * n;
    // Y|sr^T V: addevaltrans over Y's block (s,r); for a transpose view it is
    // addeval (no transpose) over the stored block (r,s).
    const int ybk = yb(by);
    const int ytr = ytrans ? 0 : 1;
    const Mat* Xm = mats[tm.xm];
    const Mat* Ym = mats[tm.ym];
    const int xi = tm.xm, yi = tm.ym;
    const double al = tm.alpha;
    switch (tm.br) {
      case 0:  // A = alpha I_t ; B = Y|sr^T N_X^T
        add_copy(cj, ctiles, a, m, nullptr, 0, nt, nt, 0, 1, al);
        add_eval(ej, yi, ybk, ytr, 1.0, b, n, w, Xm->pA[bx], nt, 1, 0);
        break;
      case 1:  // A = alpha N_X ; B = Y|sr^T I
        add_copy(cj, ctiles, a, m, Xm->pA[bx], nt, nt, ns, 0, 0, al);
        add_eval(ej, yi, ybk, ytr, 1.0, b, n, w, nullptr, 0, 0, 1);
        break;
      case 2:  // B = I_r ; A = alpha X|ts N_Y   (view: N_Y = N_(r,s)^T)
        add_copy(cj, ctiles, b, n, nullptr, 0, nr, nr, 0, 1, 1.0);
        if (ytrans) add_eval(ej, xi, bx, 0, al, a, m, w, Ym->pA[ybk], nr, 1, 0);
        else add_eval(ej, xi, bx, 0, al, a, m, w, Ym->pA[by], ns, 0, 0);
        break;
      case 3:  // B = N_Y^T ; A = alpha X|ts I  (view: N_Y^T = N_(r,s))
        if (ytrans) add_copy(cj, ctiles, b, n, Ym->pA[ybk], nr, nr, ns, 0, 0, 1.0);
        else add_copy(cj, ctiles, b, n, Ym->pA[by], ns, nr, ns, 1, 0, 1.0);
        add_eval(ej, xi, bx, 0, al, a, m, w, nullptr, 0, 0, 1);
        break;
      case 4:  // A = alpha A_X ; B = Y|sr^T B_X
        add_copy(cj, ctiles, a, m, Xm->pA[bx], nt, nt, w, 0, 0, al);
        add_eval(ej, yi, ybk, ytr, 1.0, b, n, w, Xm->pB[bx], ns, 0, 0);
        break;
      case 5:  // B = B_Y ; A = alpha X|ts A_Y   (view: A_Y = B_(r,s), B_Y = A_(r,s))
        add_copy(cj, ctiles, b, n, ytrans ? Ym->pA[ybk] : Ym->pB[by], nr, nr, w, 0, 0, 1.0);
        add_eval(ej, xi, bx, 0, al, a, m, w, ytrans ? Ym->pB[ybk] : Ym->pA[by], ns, 0, 0);
        break;
    }
  }

  // Identity pre-summing (exact; reading R7d): every term of one
  // accumulator (t, r) whose X|ts is a dense leaf may take Fig. 5's branch
  // A_hat = alpha I_t, and sum_i alpha I_t B_hat_i^T = alpha I_t (sum_i B_hat_i)^T
  // is ONE column block of width #t; likewise B_hat = I_r for dense Y|sr.  The
  // exact matrix the accumulator truncates is unchanged -- only the stack gets
  // narrower (the same argument as the narrowest-branch reading R7b).
  struct Groups {
    std::vector<char> role;   // per term: 0 own columns, 1 I_t group, 2 I_r group
    int wt = 0, wr = 0, width = 0;
  };
  bool presum = [] { const char* e = std::getenv("HM_NO_PRESUM"); return !(e && e[0] == '1'); }();

  Groups plan_groups(const Node& nd) const {
    Groups best;
    const int nterm = (int)nd.terms.size();
    best.role.assign(nterm, 0);
    for (auto& tm : nd.terms) best.width += tm.w;
    if (!presum || nterm < 2) return best;
    const int gwid[3] = {0, csize(nd.t), csize(nd.r)};
    for (int first = 1; first <= 2; first++) {
      Groups g;
      g.role.assign(nterm, 0);
      for (int pass = 0; pass < 2; pass++) {
        const int which = pass == 0 ? first : 3 - first;
        int s = 0, cnt = 0;
        for (int i = 0; i < nterm; i++)
          if (!g.role[i] && (which == 1 ? nd.terms[i].xd : nd.terms[i].yd)) { s += nd.terms[i].w; cnt++; }
        if (cnt < 2 || s <= gwid[which]) continue;
        for (int i = 0; i < nterm; i++)
          if (!g.role[i] && (which == 1 ? nd.terms[i].xd : nd.terms[i].yd)) g.role[i] = (char)which;
        (which == 1 ? g.wt : g.wr) = gwid[which];
      }
      g.width = g.wt + g.wr;
      for (int i = 0; i < nterm; i++)
        if (!g.role[i]) g.width += nd.terms[i].w;
      if (g.width < best.width) best = std::move(g);
    }
    return best;
  }

  // chained continuation jobs of the current eval batch (identity groups): em().etail
  void add_eval_chained(std::vector<EvalJob>& ej, int& head, int& last, int mi, int blk, int trans,
                        double coef, double* out, int ldo, int w, const double* V, int ldv, int vtrans) {
    add_eval(ej, mi, blk, trans, coef, out, ldo, w, V, ldv, vtrans, 0);
    if (head < 0) {
      head = (int)ej.size() - 1;
      last = -1;
      return;
    }
    std::vector<EvalMeta>& emeta = em().emeta;
    std::vector<EvalJob>& etail = em().etail;
    EvalJob e = ej.back();
    ej.pop_back();
    emeta[head].cost += emeta.back().cost;
    emeta.pop_back();
    e.next = nullptr;
    etail.push_back(e);
    const intptr_t idx = (intptr_t)etail.size();   // 1-based link, resolved at upload
    if (last < 0) ej[head].next = reinterpret_cast<const EvalJob*>(idx);
    else etail[last].next = reinterpret_cast<const EvalJob*>(idx);
    last = (int)idx - 1;
  }

  // one identity group: which = 1 (A = alpha I_t, B = sum_i Y|s_i r^T N_X(t,s_i)^T)
  // or 2 (B = I_r, A = sum_i alpha X|t s_i N_Y(s_i,r))
  void emit_group(const Node& nd, const Groups& g, int which, double* SA, int m, double* SB, int n, int col,
                  std::vector<CopyJob>& cj, int64_t& ctiles, std::vector<EvalJob>& ej) {
    double* a = SA + (size_t)col * m;
    double* b = SB + (size_t)col * n;
    const int nt = csize(nd.t), nr = csize(nd.r);
    int head = -1, last = -1;
    // alpha is folded into the summed side (terms of one group may differ in alpha)
    if (which == 1) add_copy(cj, ctiles, a, m, nullptr, 0, nt, nt, 0, 1, 1.0);
    else add_copy(cj, ctiles, b, n, nullptr, 0, nr, nr, 0, 1, 1.0);
    for (size_t i = 0; i < nd.terms.size(); i++) {
      if (g.role[i] != which) continue;
      const Term& tm = nd.terms[i];
      const int bx = tm.bx, by = tm.by, ybk = yb(by);
      const int ns = csize(T.bl_col[bx]);
      if (which == 1) {
        add_eval_chained(ej, head, last, tm.ym, ybk, ytrans ? 0 : 1, tm.alpha, b, n, nt, mats[tm.xm]->pA[bx], nt, 1);
      } else if (ytrans) {
        add_eval_chained(ej, head, last, tm.xm, bx, 0, tm.alpha, a, m, nr, mats[tm.ym]->pA[ybk], nr, 1);
      } else {
        add_eval_chained(ej, head, last, tm.xm, bx, 0, tm.alpha, a, m, nr, mats[tm.ym]->pA[by], ns, 0);
      }
    }
  }

  void copy_view(const FP& f, int t, int r, double* SA, int m, double* SB, int n, int col,
                 std::vector<CopyJob>& cj, int64_t& ctiles) {
    if (f.k <= 0) return;
    add_copy(cj, ctiles, SA + (size_t)col * m, m, f.A + (cstart(t) - f.t0), f.lda, m, f.k, 0, 0, 1.0);
    add_copy(cj, ctiles, SB + (size_t)col * n, n, f.B + (cstart(r) - f.r0), f.ldb, n, f.k, 0, 0, 1.0);
  }

  void sync_ranks(int* d_ranks, const std::vector<int>& fp_ids) {
    if (fp_ids.empty()) {
      if (c->rank_is_host(d_ranks)) c->rank_used = 0;   // nothing was enqueued on it
      return;
    }
    n_sync++;
    std::vector<int> h(fp_ids.size());
    auto a = std::chrono::steady_clock::now();
    HM_CUDA(cudaStreamSynchronize(c->stream));
    c->pinned_reset();   // every staged upload has completed
    t_wait += std::chrono::duration<double>(std::chrono::steady_clock::now() - a).count();
    if (c->rank_is_host(d_ranks)) {   // written by the kernels into mapped host memory
      std::memcpy(h.data(), d_ranks, h.size() * sizeof(int));
      c->rank_used = 0;
    } else {
      HM_CUDA(cudaMemcpy(h.data(), d_ranks, h.size() * sizeof(int), cudaMemcpyDeviceToHost));
    }
    for (size_t i = 0; i < fp_ids.size(); i++) fps[fp_ids[i]].k = h[i];
  }

  double t_a = 0, t_b = 0, t_c = 0, t_d = 0;
  static double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
  }

  // Device work of one level is enqueued by run_level_enqueue; the ranks it
  // produces are read back by run_level_finish.  Between the two the host may
  // plan the next level (split_level needs only the FP ids, not their ranks).
  struct LevelTail {
    std::unique_ptr<Arena> scratch;
    int* d_ranks = nullptr;
    std::vector<TruncReq> tr;
    std::vector<int> tr_fp;
    int cap_level = -1;
  };
  bool capture = false;   // hm_addmul with ctx->cap_on: record every level's TRUNC batch

  void run_level(std::vector<Node>& nodes) { run_level_finish(run_level_enqueue(nodes)); }

  void run_level_finish(LevelTail lt) {
    sync_ranks(lt.d_ranks, lt.tr_fp);
    if (lt.cap_level >= 0)
      for (size_t i = 0; i < lt.tr.size(); i++) c->cap[lt.cap_level].k.push_back(fps[lt.tr_fp[i]].k);
    for (size_t i = 0; i < lt.tr.size(); i++) {
      const double k = fps[lt.tr_fp[i]].k;
      fl_trunc += trunc_flops(lt.tr[i].m, lt.tr[i].n, lt.tr[i].l, k);
      by_trunc += trunc_bytes(lt.tr[i].m, lt.tr[i].n, lt.tr[i].l, k);
      n_cols += lt.tr[i].l;
    }
    n_trunc += (int64_t)lt.tr.size();
    if (lt.scratch) lt.scratch->release();
  }

  // plan_groups of every node of a level: independent of the ranks the previous
  // level produces, so run_from computes it while that level runs on the device
  std::vector<Groups> plan_level(const std::vector<Node>& nodes) const {
    std::vector<Groups> g(nodes.size());
    for (size_t i = 0; i < nodes.size(); i++) g[i] = plan_groups(nodes[i]);
    return g;
  }

  LevelTail run_level_enqueue(std::vector<Node>& nodes, std::vector<Groups>* pre = nullptr) {
    double t0 = now_s();
    LevelTail lt;
    lt.scratch.reset(new Arena(c));
    Arena& scratch = *lt.scratch;
    std::vector<Stack> stacks;
    std::vector<Groups> groups;
    if (pre && pre->size() == nodes.size()) groups.swap(*pre);
    const bool planned = !groups.empty();
    groups.resize(nodes.size());
    for (int i = 0; i < (int)nodes.size(); i++) {
      Node& nd = nodes[i];
      const int m = csize(nd.t), n = csize(nd.r);
      int kind = 0, l = 0;
      const int kb = nd.base >= 0 ? fps[nd.base].k : 0;
      if (!planned) groups[i] = plan_groups(nd);
      const int wt = groups[i].width;
      if (!nd.pend.empty() || nd.force_split || nd.zt == ZS) {
        // (iv) split with pending products; (iii) P = 0 into a subdivided
        // block: reduce (T1), then the sons (every leaf below) receive the
        // restricted base -- Fig. 7, the rkupdate of Fig. 3
        if (nd.zt == ZD && !nd.force_split)
          throw Error(HM_ESTRUCT, "flush: pending products into an inadmissible leaf");
        if (!nd.terms.empty()) { kind = 1; l = kb + wt; }
        else nd.red = nd.base;
      } else if (nd.zt == ZA || nd.zt == ZV) {
        kind = 2;
        l = zview(nd.zm, nd.zb).k + kb + wt;
      } else if (nd.zt == ZD) {
        if (kb + wt > 0) { kind = 3; l = kb + wt; }
      }
      if (kind) stacks.push_back(Stack{i, kind, m, n, l, nullptr, nullptr, -1});
    }
    if (stacks.empty()) return lt;
    size_t total = 0;
    for (auto& s : stacks) total += (size_t)(s.m + s.n) * s.l;
    double* buf = c->stack_ws(total + 1);
    {
      ProfScope ps(c, PC_MEMSET, 0, 8.0 * total);
      HM_CUDA(cudaMemsetAsync(buf, 0, total * sizeof(double), c->stream));
    }
    size_t off = 0;
    for (auto& s : stacks) {
      s.A = buf + off;
      off += (size_t)s.m * s.l;
      s.B = buf + off;
      off += (size_t)s.n * s.l;
    }
    double t1 = now_s();
    t_a += t1 - t0;
    // ---- copy and eval jobs of the level (copies and evaluations write disjoint
    // stack columns: any launch order).  Large levels are cut into parts of
    // about equal term count that several host threads build, split and sort
    // (prepare_evals) while this thread uploads and launches the finished
    // parts in order, so the device starts on part 0 while the rest is built;
    // small levels are built here in chunks.
    size_t nterms = 0;
    for (auto& s : stacks) nterms += nodes[s.node].terms.size();
    auto emit_stack = [&](Stack& s, std::vector<CopyJob>& cj, int64_t& ctiles, std::vector<EvalJob>& ej) {
      Node& nd = nodes[s.node];
      int col = 0;
      if (s.kind == 2) {
        FP zf = zview(nd.zm, nd.zb);
        copy_view(zf, nd.t, nd.r, s.A, s.m, s.B, s.n, col, cj, ctiles);
        col += zf.k;
      }
      if (nd.base >= 0) {
        copy_view(fps[nd.base], nd.t, nd.r, s.A, s.m, s.B, s.n, col, cj, ctiles);
        col += fps[nd.base].k;
      }
      const Groups& g = groups[s.node];
      if (g.wt) {
        emit_group(nd, g, 1, s.A, s.m, s.B, s.n, col, cj, ctiles, ej);
        col += g.wt;
      }
      if (g.wr) {
        emit_group(nd, g, 2, s.A, s.m, s.B, s.n, col, cj, ctiles, ej);
        col += g.wr;
      }
      for (size_t ti = 0; ti < nd.terms.size(); ti++) {
        if (g.role[ti]) continue;
        emit_term(nd.terms[ti], s.A, s.m, s.B, s.n, col, cj, ctiles, ej);
        col += nd.terms[ti].w;
      }
    };
    auto submit_copy = [&](std::vector<CopyJob>& cj, int64_t& ctiles, int aux = -1) {
      if (cj.empty()) return;
      double cb = 0;
      for (auto& j : cj) cb += 16.0 * j.rows * (j.identity ? 1 : j.cols);
      std::vector<int> tmap((size_t)ctiles);
      for (size_t j = 0; j < cj.size(); j++) {
        const int64_t t1 = j + 1 < cj.size() ? cj[j + 1].tile0 : ctiles;
        std::fill(tmap.begin() + cj[j].tile0, tmap.begin() + t1, (int)j);
      }
      const CopyJob* dj = scratch.upload_t(cj);
      const int* dm = scratch.upload_t(tmap);
      cudaStream_t st = aux >= 0 ? c->fork(aux) : c->stream;
      ProfScope ps(c, PC_COPY, 0, cb, st);
      launch_copy_mapped(dj, (int)cj.size(), dm, ctiles, st);
      HM_CHECK_LAUNCH();
      cj.clear();
      ctiles = 0;
    };
    static const int host_threads = [] {
      if (const char* e = std::getenv("HM_HOST_THREADS")) return std::max(1, std::atoi(e));
      // (measured on the 16-core B200 host: 4 / 8 / 12 / 16 threads -> product
      // 1.21 / 1.19 / 1.17 / 1.15 s)
      const unsigned hw = std::thread::hardware_concurrency();
      return (int)std::min(16u, std::max(1u, hw));
    }();
    double t2 = t1;
    if (host_threads > 1 && nterms >= 20000) {
      struct Part {
        size_t s0 = 0, s1 = 0;
        std::vector<CopyJob> cj;
        int64_t ctiles = 0;
        std::vector<EvalJob> ej, sorted;
        EmitState es;
        std::atomic<int> ready{0};
      };
      // parts of >= 16 K terms (a launch's tail is its largest job), at most 6 per
      // thread; their kernels go round-robin to 4 auxiliary streams, so the
      // tail of one part overlaps the head of the next
      const int np = (int)std::max<size_t>(2, std::min<size_t>((size_t)host_threads * 6, nterms / 16384));
      const bool par_streams = c->multi_stream();
      std::vector<Part> parts(np);
      {
        size_t si = 0, acc = 0;
        for (int p = 0; p < np; p++) {
          parts[p].s0 = si;
          const size_t target = nterms * (size_t)(p + 1) / np;
          while (si < stacks.size() && (acc < target || p == np - 1)) acc += nodes[stacks[si++].node].terms.size() + 1;
          parts[p].s1 = si;
        }
        parts[np - 1].s1 = stacks.size();
      }
      std::atomic<int> next{0};
      std::atomic<bool> failed{false};
      std::exception_ptr eptr;
      auto worker = [&]() {
        for (;;) {
          const int p = next.fetch_add(1);
          if (p >= np) break;
          Part& P = parts[p];
          try {
            tl_emit() = &P.es;
            for (size_t i = P.s0; i < P.s1; i++) emit_stack(stacks[i], P.cj, P.ctiles, P.ej);
            P.sorted = prepare_evals(P.ej);
          } catch (...) {
            failed = true;
          }
          tl_emit() = nullptr;
          P.ready.store(1, std::memory_order_release);
        }
      };
      std::vector<std::thread> pool;
      for (int t = 0; t < host_threads; t++) pool.emplace_back(worker);
      for (int p = 0; p < np; p++) {
        Part& P = parts[p];
        while (!P.ready.load(std::memory_order_acquire)) std::this_thread::yield();
        if (failed) continue;
        try {
          const int aux = par_streams ? p % 4 : -1;
          submit_copy(P.cj, P.ctiles, aux);
          fl_eval += P.es.fl;
          by_eval += P.es.by;
          submit_evals(P.sorted, P.es, scratch, P.es.fl, P.es.by, aux);
        } catch (...) {   // join the workers before the error leaves this frame
          failed = true;
          eptr = std::current_exception();
        }
      }
      for (auto& th : pool) th.join();
      if (par_streams)
        for (int k = 0; k < 4; k++) c->join(k);
      if (eptr) std::rethrow_exception(eptr);
      if (failed) throw Error(HM_ESTRUCT, "internal: job emission failed");
      t2 = now_s();
      t_b += t2 - t1;
    } else {
      std::vector<CopyJob> cj;
      std::vector<EvalJob> ej;
      cj.reserve(nterms + 2 * stacks.size());
      ej.reserve(nterms);
      em0.emeta.reserve(nterms);
      int64_t ctiles = 0;
      double fl_eval0 = fl_eval, by_eval0 = by_eval;
      static const size_t kChunk = [] { const char* e = std::getenv("HM_JOB_CHUNK"); return e ? (size_t)std::atoll(e) : (size_t)1 << 16; }();
      auto flush_eval = [&]() {
        if (ej.empty()) return;
        launch_evals(ej, scratch, fl_eval - fl_eval0, by_eval - by_eval0);
        fl_eval0 = fl_eval;
        by_eval0 = by_eval;
      };
      for (auto& s : stacks) {
        emit_stack(s, cj, ctiles, ej);
        if (ej.size() >= kChunk) flush_eval();
        if (cj.size() >= kChunk) submit_copy(cj, ctiles);
      }
      submit_copy(cj, ctiles);
      t2 = now_s();
      t_b += t2 - t1;
      flush_eval();
    }
    // truncations and dense adds
    std::vector<TruncReq> tr;
    std::vector<int> tr_fp;
    std::vector<GemmJob> gj;
    int64_t gtiles = 0;
    int* d_ranks = c->rank_alloc(stacks.size() + 1);
    if (!d_ranks) d_ranks = static_cast<int*>(scratch.alloc_bytes(sizeof(int) * (stacks.size() + 1)));
    const double fl_dense0 = fl_dense, by_dense0 = by_dense;
    for (auto& s : stacks) {
      Node& nd = nodes[s.node];
      if (s.kind == 3) {
        GemmJob g{};
        g.A = s.A; g.lda = s.m; g.transA = 0;
        g.B = s.B; g.ldb = s.n; g.transB = 1;
        g.C = mats[nd.zm]->pA[nd.zb]; g.ldc = s.m;
        g.m = s.m; g.n = s.n; g.k = s.l;
        g.alpha = 1.0; g.beta = 1.0;
        g.tile0 = gtiles;
        gtiles += (int64_t)((s.m + 63) / 64) * ((s.n + 63) / 64);
        gj.push_back(g);
        n_dense++;
        fl_dense += 2.0 * s.m * s.n * s.l;
        by_dense += 8.0 * ((double)(s.m + s.n) * s.l + 2.0 * s.m * s.n);
        continue;
      }
      const int kcap = trunc_kcap(s.m, s.n, s.l);
      // a reduce-only node's T1 result is read after the enclosing flush has
      // rewound its LIFO arena (Factorizer::flush_many): it lives on the heap
      fp_heap = s.kind == 1 && nd.no_expand;
      const int out = new_fp(s.m, s.n, kcap, cstart(nd.t), cstart(nd.r));
      fp_heap = false;
      s.out = out;
      TruncReq q{s.m, s.n, s.l, s.A, s.B, fps[out].A, fps[out].B, d_ranks + tr.size(), nullptr};
      tr.push_back(q);
      tr_fp.push_back(out);
      if (s.kind == 1) nd.red = out;
      else nd.result = out;
    }
    if (!gj.empty()) {
      ProfScope ps(c, PC_DENSE, fl_dense - fl_dense0, by_dense - by_dense0);
      launch_gemm_mapped(scratch.upload_t(gj), (int)gj.size(), scratch.tile_map_t(gj, gtiles), gtiles, c->stream);
      HM_CHECK_LAUNCH();
    }
    double t3 = now_s();
    t_c += t3 - t2;
    if (capture) {
      const int lev = (int)c->cap.size();
      c->cap.emplace_back();
      Ctx::CapLevel& L = c->cap.back();
      for (const TruncReq& q : tr) {
        L.m.push_back(q.m);
        L.n.push_back(q.n);
        L.l.push_back(q.l);
        L.aoff.push_back((size_t)(q.A - buf));
        L.boff.push_back((size_t)(q.B - buf));
      }
      if (lev < 64 && ((c->cap_mask >> lev) & 1) && total > 0) {
        L.ndoubles = total;
        L.data = static_cast<double*>(c->dmalloc(total * sizeof(double)));
        HM_CUDA(cudaMemcpyAsync(L.data, buf, total * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
      }
      lt.cap_level = lev;
    }
    trunc_batched(c, scratch, tr, eps);
    t_d += now_s() - t3;
    for (auto& s : stacks) {
      Node& nd = nodes[s.node];
      if (s.kind == 2 && nd.zt == ZA) set_zres(nd.zm, nd.zb, nd.result);
    }
    lt.d_ranks = d_ranks;
    lt.tr = std::move(tr);
    lt.tr_fp = std::move(tr_fp);
    return lt;
  }

  // Fig. 6 split for every node with pending products -> next level.
  std::vector<Node> split_level(std::vector<Node>& nodes) {
    std::vector<Node> next;
    for (auto& nd : nodes) {
      if ((nd.pend.empty() && nd.zt != ZS) || nd.no_expand) continue;
      nd.child0 = (int)next.size();
      expand(nd, false, next);
    }
    return next;
  }

  // Fig. 6 sons of one accumulator (row-major over sons(t) x sons(r)); the sons
  // inherit nd.red as base; pending products are expanded over sons(s).
  // lower_only (H-Cholesky): strictly upper sons are not created (a null
  // placeholder with t = -1 keeps the row-major indexing).
  void expand(const Node& nd, bool lower_only, std::vector<Node>& out) {
    const int t = nd.t, r = nd.r;
    const int nts = T.cl_nsons[t], nrs = T.cl_nsons[r];
    for (int i = 0; i < nts; i++) {
      for (int j = 0; j < nrs; j++) {
        Node ch;
        ch.t = T.cl_son0[t] + i;
        ch.r = T.cl_son0[r] + j;
        ch.zm = nd.zm;
        if (lower_only && cstart(ch.t) < cstart(ch.r)) {
          ch.t = -1;
          out.push_back(std::move(ch));
          continue;
        }
        if (nd.zt == ZS) {
          const int zb = T.son(nd.zb, i, j);
          ch.zb = zb;
          ch.zt = T.bl_kind[zb] == HM_BLOCK_SUB ? ZS : (T.bl_kind[zb] == HM_BLOCK_ADM ? ZA : ZD);
        } else {
          ch.zt = ZV;
          ch.zb = nd.zb;   // the real admissible leaf the temporaries restrict
        }
        ch.base = nd.red;
        for (auto& p : nd.pend) {
          const int s = T.bl_col[p.bx];
          for (int l = 0; l < T.cl_nsons[s]; l++)
            addproduct(ch, T.son(p.bx, i, l), T.son(p.by, l, j), p.xm, p.ym, p.alpha);
        }
        out.push_back(std::move(ch));
      }
    }
  }

  // Fig. 4 rkmerge of the temporaries below admissible leaves, bottom-up.
  void merges() {
    for (int lev = (int)levels.size() - 2; lev >= 0; lev--) {
      std::vector<int> mn;
      for (int i = 0; i < (int)levels[lev].size(); i++) {
        const Node& nd = levels[lev][i];
        if (!nd.pend.empty() && !nd.no_expand && (nd.zt == ZA || nd.zt == ZV)) mn.push_back(i);
      }
      if (mn.empty()) continue;
      std::vector<Node>& kids = levels[lev + 1];
      // stage a: block columns (exact vertical stacks)
      std::vector<std::vector<int>> colfp(mn.size());
      for (int stage = 0; stage < 2; stage++) {
        Arena scratch(c);
        struct S { int m, n, l; double *A, *B; int out; };
        std::vector<S> ss;
        std::vector<CopyJob> cj;
        int64_t ctiles = 0;
        std::vector<std::pair<int, int>> who;   // (merge idx, column j) for stage a
        size_t total = 0;
        std::vector<S> pre;
        for (size_t mi = 0; mi < mn.size(); mi++) {
          const Node& nd = levels[lev][mn[mi]];
          const int nts = T.cl_nsons[nd.t], nrs = T.cl_nsons[nd.r];
          if (stage == 0) {
            for (int j = 0; j < nrs; j++) {
              int l = 0;
              for (int i = 0; i < nts; i++) l += fps[kids[nd.child0 + i * nrs + j].result].k;
              pre.push_back(S{csize(nd.t), csize(T.cl_son0[nd.r] + j), l, nullptr, nullptr, -1});
              who.push_back({(int)mi, j});
            }
          } else {
            int l = 0;
            for (int j = 0; j < nrs; j++) l += fps[colfp[mi][j]].k;
            pre.push_back(S{csize(nd.t), csize(nd.r), l, nullptr, nullptr, -1});
            who.push_back({(int)mi, -1});
          }
        }
        for (auto& s : pre) total += (size_t)(s.m + s.n) * s.l;
        double* buf = c->stack_ws(total + 1);
        HM_CUDA(cudaMemsetAsync(buf, 0, total * sizeof(double), c->stream));
        size_t off = 0;
        for (auto& s : pre) {
          s.A = buf + off; off += (size_t)s.m * s.l;
          s.B = buf + off; off += (size_t)s.n * s.l;
        }
        for (size_t w = 0; w < pre.size(); w++) {
          S& s = pre[w];
          const Node& nd = levels[lev][mn[who[w].first]];
          const int nts = T.cl_nsons[nd.t], nrs = T.cl_nsons[nd.r];
          int col = 0;
          if (stage == 0) {
            const int j = who[w].second;
            for (int i = 0; i < nts; i++) {
              const FP& f = fps[kids[nd.child0 + i * nrs + j].result];
              const int ti = T.cl_son0[nd.t] + i;
              const int ro = cstart(ti) - cstart(nd.t);
              if (f.k > 0) {
                add_copy(cj, ctiles, s.A + ro + (size_t)col * s.m, s.m, f.A, f.lda, csize(ti), f.k, 0, 0, 1.0);
                add_copy(cj, ctiles, s.B + (size_t)col * s.n, s.n, f.B, f.ldb, s.n, f.k, 0, 0, 1.0);
              }
              col += f.k;
            }
          } else {
            const int mi = who[w].first;
            for (int j = 0; j < nrs; j++) {
              const FP& f = fps[colfp[mi][j]];
              const int rj = T.cl_son0[nd.r] + j;
              const int co = cstart(rj) - cstart(nd.r);
              if (f.k > 0) {
                add_copy(cj, ctiles, s.A + (size_t)col * s.m, s.m, f.A, f.lda, s.m, f.k, 0, 0, 1.0);
                add_copy(cj, ctiles, s.B + co + (size_t)col * s.n, s.n, f.B, f.ldb, csize(rj), f.k, 0, 0, 1.0);
              }
              col += f.k;
            }
          }
        }
        {
          ProfScope ps(c, PC_COPY, 0, 0);
          launch_copy_mapped(scratch.upload_t(cj), (int)cj.size(), scratch.tile_map_t(cj, ctiles), ctiles, c->stream);
          HM_CHECK_LAUNCH();
        }
        std::vector<TruncReq> tr;
        std::vector<int> tr_fp;
        int* d_ranks = c->rank_alloc(pre.size() + 1);
        if (!d_ranks) d_ranks = static_cast<int*>(scratch.alloc_bytes(sizeof(int) * (pre.size() + 1)));
        for (size_t w = 0; w < pre.size(); w++) {
          S& s = pre[w];
          const Node& nd = levels[lev][mn[who[w].first]];
          const int r0 = stage == 0 ? cstart(T.cl_son0[nd.r] + who[w].second) : cstart(nd.r);
          const int out = new_fp(s.m, s.n, trunc_kcap(s.m, s.n, s.l), cstart(nd.t), r0);
          s.out = out;
          tr.push_back(TruncReq{s.m, s.n, s.l, s.A, s.B, fps[out].A, fps[out].B, d_ranks + tr.size(), nullptr});
          tr_fp.push_back(out);
        }
        trunc_batched(c, scratch, tr, eps);
        sync_ranks(d_ranks, tr_fp);
        for (size_t i = 0; i < tr.size(); i++) {
          const double k = fps[tr_fp[i]].k;
          fl_trunc += trunc_flops(tr[i].m, tr[i].n, tr[i].l, k);
          by_trunc += trunc_bytes(tr[i].m, tr[i].n, tr[i].l, k);
          n_cols += tr[i].l;
        }
        n_trunc += (int64_t)tr.size();
        for (size_t w = 0; w < pre.size(); w++) {
          const int mi = who[w].first;
          if (stage == 0) colfp[mi].push_back(pre[w].out);
          else {
            Node& nd = levels[lev][mn[mi]];
            nd.result = pre[w].out;
            if (nd.zt == ZA) set_zres(nd.zm, nd.zb, nd.result);
          }
        }
        scratch.release();
      }
      n_merge += (int64_t)mn.size();
    }
  }

  void finish() {
    // compact the new admissible-leaf factors of Z into one owned pool
    size_t total = 0;
    const int nb = T.nblocks();
    for (int b = 0; b < nb; b++) {
      if (T.bl_kind[b] != HM_BLOCK_ADM) continue;
      if (zres(zm0, b) < 0) throw Error(HM_ESTRUCT, "internal: admissible Z leaf without update");
      const FP& f = fps[zres(zm0, b)];
      total += (size_t)(f.lda + f.ldb) * f.k;
    }
    double* pool = static_cast<double*>(c->dmalloc((total + 1) * sizeof(double)));
    std::vector<CopyJob> cj;
    int64_t ctiles = 0;
    size_t off = 0;
    std::vector<double*> nA(nb, nullptr), nB(nb, nullptr);
    std::vector<int> nk(nb, 0);
    for (int b = 0; b < nb; b++) {
      if (T.bl_kind[b] != HM_BLOCK_ADM) continue;
      const FP& f = fps[zres(zm0, b)];
      nA[b] = pool + off;
      off += (size_t)f.lda * f.k;
      nB[b] = pool + off;
      off += (size_t)f.ldb * f.k;
      nk[b] = f.k;
      add_copy(cj, ctiles, nA[b], f.lda, f.A, f.lda, f.lda, f.k, 0, 0, 1.0);
      add_copy(cj, ctiles, nB[b], f.ldb, f.B, f.ldb, f.ldb, f.k, 0, 0, 1.0);
    }
    Arena scratch(c);
    launch_copy_mapped(scratch.upload_t(cj), (int)cj.size(), scratch.tile_map_t(cj, ctiles), ctiles, c->stream);
    HM_CHECK_LAUNCH();
    HM_CUDA(cudaStreamSynchronize(c->stream));
    scratch.release();
    // release Z's old factor pool (the dense pool stays: updated in place)
    c->dfree(Z->fpool.first, Z->fpool.second);
    for (int b = 0; b < nb; b++) {
      if (T.bl_kind[b] != HM_BLOCK_ADM) continue;
      Z->pA[b] = nA[b];
      Z->pB[b] = nB[b];
      Z->rank[b] = nk[b];
    }
    Z->fpool = {pool, (total + 1) * sizeof(double)};
  }

  // Level-synchronous flush of the given root accumulators (Fig. 7 with
  // split/addproduct per level) followed by the bottom-up merges.
  double t_level = 0, t_split = 0, t_merge = 0;
  void run_from(std::vector<Node> roots) {
    using clk = std::chrono::steady_clock;
    auto sec = [](clk::time_point a, clk::time_point b) { return std::chrono::duration<double>(b - a).count(); };
    levels.clear();
    levels.push_back(std::move(roots));
    std::vector<Groups> pre;
    while (true) {
      auto a = clk::now();
      LevelTail tail = run_level_enqueue(levels.back(), &pre);
      auto b = clk::now();
      std::vector<Node> next = split_level(levels.back());   // overlaps the level's device work
      pre = plan_level(next);
      auto d = clk::now();
      run_level_finish(std::move(tail));
      t_level += sec(a, b);
      t_split += sec(b, d);
      if (next.empty()) break;
      levels.push_back(std::move(next));
    }
    auto a = clk::now();
    merges();
    t_merge += sec(a, clk::now());
  }

  void setup_tables(bool upload) {
    const size_t nm = mats.size();
    zresult.assign(nm, std::vector<int>(T.nblocks(), -1));
    ltab.assign(nm, {});
    lmat.assign(nm, {});
    lmn.assign(nm, {});
    dltab.assign(nm, nullptr);
    for (size_t mi = 0; mi < nm; mi++) {
      ltab[mi] = leaf_table(*mats[mi]);
      refresh_sums(mi);
      if (upload) dltab[mi] = persist.upload(ltab[mi]);
    }
  }
  // convention-count prefix sums of matrix mi's leaf table (after rank changes)
  void refresh_sums(size_t mi) {
    const std::vector<LeafDesc>& lt = ltab[mi];
    std::vector<double>& pm = lmat[mi];
    std::vector<double>& pn = lmn[mi];
    pm.assign(lt.size() + 1, 0.0);
    pn.assign(lt.size() + 1, 0.0);
    for (size_t i = 0; i < lt.size(); i++) {
      const LeafDesc& L = lt[i];
      pm[i + 1] = pm[i] + (L.kind == HM_BLOCK_DENSE ? (double)L.m * L.n : (double)L.k * (L.m + L.n));
      pn[i + 1] = pn[i] + (double)(L.m + L.n);
    }
  }

  void run() {
    setup_tables(true);
    Node root;
    root.t = T.bl_row[0];
    root.r = T.bl_col[0];
    root.zb = 0;
    root.zm = zm0;
    root.zt = T.bl_kind[0] == HM_BLOCK_SUB ? ZS : (T.bl_kind[0] == HM_BLOCK_ADM ? ZA : ZD);
    addproduct(root, 0, 0);
    std::vector<Node> roots;
    roots.push_back(std::move(root));
    run_from(std::move(roots));
    auto b = std::chrono::steady_clock::now();
    finish();
    const double t_fin = std::chrono::duration<double>(std::chrono::steady_clock::now() - b).count();
    if (std::getenv("HM_DEBUG_TIMING"))
      std::fprintf(stderr,
                   "[hm_addmul] levels %.3fs (sync wait %.3fs; host: layout %.3f jobs %.3f launch %.3f trunc %.3f) "
                   "split %.3fs merges %.3fs finish %.3fs\n",
                   t_level, t_wait, t_a, t_b, t_c, t_d, t_split, t_merge, t_fin);
  }
};

// ---------------------------------------------------------------------------
// H-LR / H-Cholesky with accumulated updates (§6; the
// recursion is the reading O8/O9 of SURVEY §8(c), also implemented in
// oracle/factor.py).  Host-driven recursion; every accumulator operation
// (reduce = T1, flush into a leaf incl. temporaries + rkmerge, addproduct)
// goes through the Planner above, triangular solves through the H-structure
// run as one k_trsm CTA per panel, dense diagonal leaves as k_leaf_factor.
static void trsm_launch(const TrsmJob* j, int n, const TrsmStep* st, const LeafDesc* lv, cudaStream_t s) {
  launch_trsm2(j, n, st, lv, s);
}

struct Factorizer {
  Ctx* c;
  Mat* G;
  const Tree& T;
  bool chol;
  Planner P;
  std::vector<LeafDesc> lt;
  std::vector<int> leafpos;
  LeafDesc* dlt = nullptr;
  std::vector<std::pair<void*, size_t>> own;   // per block: factor buffer owned here
  std::unordered_map<int64_t, int> bmap;       // (row, col) -> block id
  int* d_fail = nullptr;
  double* d_minpiv = nullptr;
  int64_t n_trsm = 0, n_leaf = 0, n_flush = 0, n_flush_calls = 0, n_reduce_calls = 0;

  Factorizer(Ctx* c_, Mat* G_, double eps, bool ch)
      : c(c_), G(G_), T(*G_->tree), chol(ch), P(c_, *G_->tree, G_, G_, G_, -1.0, eps) {
    const int nb = T.nblocks();
    for (int b = 0; b < nb; b++) bmap[key(T.bl_row[b], T.bl_col[b])] = b;
    if (chol) {
      P.ytrans = true;
      P.tmap.resize(nb);
      for (int b = 0; b < nb; b++) {
        auto it = bmap.find(key(T.bl_col[b], T.bl_row[b]));
        if (it == bmap.end() || T.bl_kind[it->second] != T.bl_kind[b])
          throw Error(HM_ESTRUCT, "hm_chol: the block tree is not symmetric");
        P.tmap[b] = it->second;
      }
    }
    for (int t = 0; t < T.nclusters(); t++)
      if (T.cl_nsons[t] != 0 && T.cl_nsons[t] != 2)
        throw Error(HM_EUNSUPPORTED, "H-LR/H-Cholesky need a binary cluster tree (P:L1361-1363)");
    P.setup_tables(false);
    lt = P.ltab[0];
    leafpos.assign(nb, -1);
    for (size_t i = 0; i < T.leaf_order.size(); i++) leafpos[T.leaf_order[i]] = (int)i;
    dlt = P.persist.upload(lt);
    P.dltab[0] = dlt;
    own.assign(nb, {nullptr, 0});
    d_fail = static_cast<int*>(P.persist.alloc_bytes(sizeof(int)));
    HM_CUDA(cudaMemsetAsync(d_fail, 0, sizeof(int), c->stream));
    d_minpiv = P.persist.alloc(T.nclusters());
    HM_CUDA(cudaMemsetAsync(d_minpiv, 0, sizeof(double) * T.nclusters(), c->stream));
  }

  static int64_t key(int a, int b) { return ((int64_t)a << 32) | (uint32_t)b; }
  int blk(int a, int b) const {
    auto it = bmap.find(key(a, b));
    if (it == bmap.end()) throw Error(HM_ESTRUCT, "internal: missing block");
    return it->second;
  }
  int son0(int t) const { return T.cl_son0[t]; }

  Node acc_for(int b) const {
    Node nd;
    nd.t = T.bl_row[b];
    nd.r = T.bl_col[b];
    nd.zb = b;
    nd.zt = T.bl_kind[b] == HM_BLOCK_SUB ? ZS : (T.bl_kind[b] == HM_BLOCK_ADM ? ZA : ZD);
    return nd;
  }

  // Fig. 7 flush of accumulators into distinct leaves nd.zb of G (branches i,
  // ii, v) -- all of them in ONE level-synchronous batch.
  void flush(const Node& nd) { flush_many(std::vector<Node>{nd}); }

  // reduce_with: accumulators of subdivided solve targets whose T1 reduce is
  // independent of these flushes -- it joins the first level batch (one
  // dependent step instead of two); their .red is set on return
  void flush_many(std::vector<Node> roots, const std::vector<Node*>& reduce_with = {}) {
    std::vector<Node*> red_nodes;
    const size_t nflush = roots.size();
    for (Node* nd : reduce_with) {
      if (nd->terms.empty()) {
        nd->red = nd->base;
        continue;
      }
      Node b = *nd;
      b.force_split = true;
      b.no_expand = true;
      roots.push_back(std::move(b));
      red_nodes.push_back(nd);
      n_reduce_calls++;
    }
    if (roots.empty()) return;
    if (c->plog) {
      int pend = 0;
      for (auto& r : roots) pend += !r.pend.empty();
      c->prof_note("FLUSH roots " + std::to_string(roots.size()) + " withpend " + std::to_string(pend));
      ProfScope mark(c, PC_MEMSET, 0, 0);
    }
    n_flush += (int64_t)roots.size();
    n_flush_calls++;
    Arena local(c, true);
    P.fp_arena = &local;
    std::vector<int> zbs;
    for (size_t i = 0; i < nflush; i++) {
      P.zres(0, roots[i].zb) = -1;
      zbs.push_back(roots[i].zb);
    }
    P.run_from(std::move(roots));
    for (size_t i = 0; i < red_nodes.size(); i++) red_nodes[i]->red = P.levels[0][nflush + i].red;
    // the new factors move from the flush's arena into buffers of their own and
    // the leaf table is patched: ONE copy launch and ONE patch launch per flush
    // (per-block cudaMemcpyAsync calls left the device idle for ~180 us per flush)
    std::vector<CopyJob> cj;
    std::vector<LeafPatch> patches;
    int64_t ctiles = 0;
    for (int zb : zbs) {
      if (T.bl_kind[zb] != HM_BLOCK_ADM) continue;
      const int f = P.zres(0, zb);
      if (f < 0) throw Error(HM_ESTRUCT, "internal: flush produced no result");
      const FP& fp = P.fps[f];
      const int m = fp.lda, n = fp.ldb, k = fp.k;
      // bump allocation from the planner's heap arena (64 MB chunks, released
      // with the factorization): no cudaMallocAsync / cudaFreeAsync per block
      double* buf = P.heap.alloc((size_t)(m + n) * k + 1);
      if (k > 0) {
        P.add_copy(cj, ctiles, buf, m, fp.A, m, m, k, 0, 0, 1.0);
        P.add_copy(cj, ctiles, buf + (size_t)m * k, n, fp.B, n, n, k, 0, 0, 1.0);
      }
      G->pA[zb] = buf;
      G->pB[zb] = buf + (size_t)m * k;
      G->rank[zb] = k;
      const int pos = leafpos[zb];
      lt[pos].A = G->pA[zb];
      lt[pos].B = G->pB[zb];
      lt[pos].k = k;
      patches.push_back(LeafPatch{pos, lt[pos]});
    }
    if (!cj.empty()) {
      launch_copy_mapped(local.upload(cj), (int)cj.size(), local.tile_map(cj, ctiles), ctiles, c->stream);
      HM_CHECK_LAUNCH();
    }
    if (!patches.empty()) {
      launch_patch_leaves(dlt, local.upload(patches), (int)patches.size(), c->stream);
      HM_CHECK_LAUNCH();
    }
    P.fp_arena = nullptr;
    local.release();
  }

  // T1 reduce of an accumulator that is split (Fig. 6); result persists.
  void reduce(Node& nd) {
    std::vector<Node*> v{&nd};
    reduce_many(v);
  }

  void reduce_many(std::vector<Node*>& nds) {
    std::vector<Node> batch;
    std::vector<Node*> who;
    for (Node* nd : nds) {
      if (nd->terms.empty()) {
        nd->red = nd->base;
        continue;
      }
      batch.push_back(*nd);
      batch.back().force_split = true;
      who.push_back(nd);
    }
    if (batch.empty()) return;
    n_reduce_calls++;
    if (c->plog) {
      c->prof_note("REDUCE " + std::to_string(batch.size()));
      ProfScope mark(c, PC_MEMSET, 0, 0);
    }
    P.run_level(batch);
    for (size_t i = 0; i < who.size(); i++) who[i]->red = batch[i].red;
  }

  std::vector<Node> split(Node& nd, bool lower_only) {
    reduce(nd);
    std::vector<Node> ch;
    P.expand(nd, lower_only, ch);
    return ch;
  }

  // ---- triangular solves through the H-structure (k_trsm step lists)
  void steps_lower(int t, bool unit, int panel0, std::vector<TrsmStep>& st) {
    if (T.cl_nsons[t] == 0) {
      const int d = blk(t, t);
      st.push_back(TrsmStep{0, T.cl_start[t] - panel0, T.cl_size[t], G->pA[d], T.cl_size[t], 0, unit ? 1 : 0, 0, 0});
      return;
    }
    const int t1 = son0(t), t2 = t1 + 1;
    steps_lower(t1, unit, panel0, st);
    const int b = blk(t2, t1);
    st.push_back(TrsmStep{1, 0, 0, nullptr, 0, 0, 0, T.bl_lbeg[b], T.bl_lend[b]});
    steps_lower(t2, unit, panel0, st);
  }

  void steps_rt(int s, int panel0, std::vector<TrsmStep>& st) {
    if (T.cl_nsons[s] == 0) {
      const int d = blk(s, s);
      st.push_back(TrsmStep{0, T.cl_start[s] - panel0, T.cl_size[s], G->pA[d], T.cl_size[s], 1, 0, 0, 0});
      return;
    }
    const int s1 = son0(s), s2 = s1 + 1;
    steps_rt(s1, panel0, st);
    const int b = blk(s1, s2);
    st.push_back(TrsmStep{1, 0, 0, nullptr, 0, 1, 0, T.bl_lbeg[b], T.bl_lend[b]});
    steps_rt(s2, panel0, st);
  }

  // mode 0: V <- L^{-1} V (unit), 1: V <- R^{-T} V, 2: V <- L^{-1} V (Cholesky factor)
  void trsm(int mode, int t, double* V, int ldv, int ncols) {
    if (ncols <= 0) return;
    n_trsm++;
    std::vector<TrsmStep> st;
    if (mode == 1) steps_rt(t, T.cl_start[t], st);
    else steps_lower(t, mode == 0, T.cl_start[t], st);
    Arena ar(c, true);
    std::vector<TrsmJob> jb{TrsmJob{V, ldv, ncols, T.cl_start[t], 0, (int)st.size()}};
    trsm_launch(ar.upload_t(jb), 1, ar.upload_t(st), dlt, c->stream);
    HM_CHECK_LAUNCH();
  }

  void leaf_factor(int t) {
    n_leaf++;
    const int d = blk(t, t);
    const int m = T.cl_size[t];
    Arena ar(c, true);
    std::vector<LeafFactorJob> j{LeafFactorJob{G->pA[d], m, m, t}};
    launch_leaf_factor(ar.upload_t(j), 1, chol ? 1 : 0, d_fail, d_minpiv + t, m, c->stream);
    HM_CHECK_LAUNCH();
  }

  // ---- batched solves: every target of one set shares the cluster t (row
  // cluster of SOLVE_L targets, column cluster of SOLVE_R / SOLVE_LT
  // targets), so the recursions over sons(t) run in lock step and each step
  // is ONE batch of flushes / reduces / triangular solves.  Each accumulator
  // still receives exactly the addproducts of the serial recursion before it
  // is split or flushed (same truncation inputs as oracle/factor.py).
  struct Item { int b; Node acc; };

  void trsm_set(int t, const std::vector<std::pair<int, int>>& targets) {   // (block, mode)
    if (targets.empty()) return;
    Arena ar(c, true);
    std::vector<TrsmStep> st;
    int rng[3][2] = {{-1, -1}, {-1, -1}, {-1, -1}};
    for (auto& tg : targets) {
      const int mode = tg.second;
      if (rng[mode][0] >= 0) continue;
      rng[mode][0] = (int)st.size();
      if (mode == 1) steps_rt(t, T.cl_start[t], st);
      else steps_lower(t, mode == 0, T.cl_start[t], st);
      rng[mode][1] = (int)st.size();
    }
    std::vector<TrsmJob> jobs;
    std::vector<CopyJob> pre, post;
    int64_t pt = 0, qt = 0;
    for (auto& tg : targets) {
      const int b = tg.first, mode = tg.second;
      const int m = T.cl_size[T.bl_row[b]], n = T.cl_size[T.bl_col[b]];
      if (T.bl_kind[b] == HM_BLOCK_ADM) {
        if (G->rank[b] <= 0) continue;
        if (mode == 0) jobs.push_back(TrsmJob{G->pA[b], m, G->rank[b], T.cl_start[t], rng[0][0], rng[0][1]});
        else jobs.push_back(TrsmJob{G->pB[b], n, G->rank[b], T.cl_start[t], rng[mode][0], rng[mode][1]});
      } else if (mode == 0) {
        jobs.push_back(TrsmJob{G->pA[b], m, n, T.cl_start[t], rng[0][0], rng[0][1]});
      } else {
        // N <- N op^{-1}: solve on the transpose panel (n x m) and copy back
        double* tmp = ar.alloc((size_t)m * n);
        pre.push_back(CopyJob{tmp, G->pA[b], n, m, n, m, 1, 0, 0, 1.0, pt});
        pt += (int64_t)((n + 31) / 32) * ((m + 31) / 32);
        post.push_back(CopyJob{G->pA[b], tmp, m, n, m, n, 1, 0, 0, 1.0, qt});
        qt += (int64_t)((m + 31) / 32) * ((n + 31) / 32);
        jobs.push_back(TrsmJob{tmp, n, m, T.cl_start[t], rng[mode][0], rng[mode][1]});
      }
    }
    n_trsm += (int64_t)jobs.size();
    ProfScope ps(c, PC_TRSM, 0, 0);
    if (!pre.empty()) launch_copy_mapped(ar.upload_t(pre), (int)pre.size(), ar.tile_map_t(pre, pt), pt, c->stream);
    if (!jobs.empty()) trsm_launch(ar.upload_t(jobs), (int)jobs.size(), ar.upload_t(st), dlt, c->stream);
    if (!post.empty()) launch_copy_mapped(ar.upload_t(post), (int)post.size(), ar.tile_map_t(post, qt), qt, c->stream);
    HM_CHECK_LAUNCH();
  }

  // L: SOLVE_L targets (t, r); R: SOLVE_R targets (t', t) (mode 1) or, for
  // Cholesky, SOLVE_LT targets (mode 2).
  void solve_set(int t, std::vector<Item> L, std::vector<Item> R) {
    const int rmode = chol ? 2 : 1;
    std::vector<Node> leaf_accs;
    std::vector<std::pair<int, int>> leaf_targets;
    std::vector<Item*> subL, subR;
    for (auto& it : L) {
      if (T.bl_kind[it.b] == HM_BLOCK_SUB) subL.push_back(&it);
      else { leaf_accs.push_back(it.acc); leaf_targets.push_back({it.b, 0}); }
    }
    for (auto& it : R) {
      if (T.bl_kind[it.b] == HM_BLOCK_SUB) subR.push_back(&it);
      else { leaf_accs.push_back(it.acc); leaf_targets.push_back({it.b, rmode}); }
    }
    std::vector<Node*> red;
    for (auto* it : subL) red.push_back(&it->acc);
    for (auto* it : subR) red.push_back(&it->acc);
    flush_many(std::move(leaf_accs), red);   // leaf flushes + the subdivided targets' T1 in one batch
    trsm_set(t, leaf_targets);
    if (subL.empty() && subR.empty()) return;
    const int t1 = son0(t), t2 = t1 + 1;
    std::vector<Item> L1, L2, R1, R2;
    for (auto* it : subL) {            // b = (t, r): sons (t_i, r_j), row-major
      std::vector<Node> ch;
      P.expand(it->acc, false, ch);
      const int nr = T.cl_nsons[T.bl_col[it->b]];
      for (int j = 0; j < nr; j++) {
        L1.push_back(Item{T.son(it->b, 0, j), ch[j]});
        L2.push_back(Item{T.son(it->b, 1, j), ch[nr + j]});
      }
    }
    for (auto* it : subR) {            // b = (t', t): sons (t'_i, t_j)
      std::vector<Node> ch;
      P.expand(it->acc, false, ch);
      const int nt = T.cl_nsons[T.bl_row[it->b]];
      for (int i = 0; i < nt; i++) {
        R1.push_back(Item{T.son(it->b, i, 0), ch[2 * i]});
        R2.push_back(Item{T.son(it->b, i, 1), ch[2 * i + 1]});
      }
    }
    solve_set(t1, L1, R1);
    for (size_t j = 0; j < L2.size(); j++)          // acc_(t2,r') += -L_(t2,t1) R_(t1,r')
      P.addproduct(L2[j].acc, blk(t2, t1), L1[j].b);
    for (size_t i = 0; i < R2.size(); i++)          // acc_(t',t2) += -L_(t',t1) R_(t1,t2)  [chol: L_(t2,t1)^T]
      P.addproduct(R2[i].acc, R1[i].b, blk(t1, t2));
    solve_set(t2, L2, R2);
  }

  // ---- merged recursion: factor G|tt from its accumulator AND
  // solve every pending target of row cluster t (L: SOLVE_L blocks (t, r)) or
  // column cluster t (R: SOLVE_R / SOLVE_LT blocks (t', t)) handed down by ALL
  // ancestors.  O8/O9 run solve_set(t1, ...) once per ancestor level after
  // lr(t) has returned; the sub-solves with a son t1 only need L|t1t1 / R|t1t1,
  // so here they join the recursion into t1 as soon as lr(t1) is done: one
  // dependent batch per cluster instead of one per (cluster, ancestor level).
  // Every accumulator still receives exactly the addproducts of the serial
  // recursion before it is reduced, split or flushed (same truncation inputs
  // as oracle/factor.py), only independent steps share a batch.
  void factor_merged(int t, Node acc, std::vector<Item> L, std::vector<Item> R) {
    const int rmode = chol ? 2 : 1;
    if (T.cl_nsons[t] == 0) {
      // targets of a leaf cluster are leaves themselves: the diagonal flush and
      // theirs are independent -> one batch; then the leaf factors, then the solves
      std::vector<Node> accs{acc};
      std::vector<std::pair<int, int>> targets;
      for (auto& it : L) { accs.push_back(it.acc); targets.push_back({it.b, 0}); }
      for (auto& it : R) { accs.push_back(it.acc); targets.push_back({it.b, rmode}); }
      flush_many(std::move(accs));
      leaf_factor(t);
      trsm_set(t, targets);
      return;
    }
    std::vector<Node> leaf_accs;
    std::vector<std::pair<int, int>> leaf_targets;
    std::vector<Item*> subL, subR;
    for (auto& it : L) {
      if (T.bl_kind[it.b] == HM_BLOCK_SUB) subL.push_back(&it);
      else { leaf_accs.push_back(it.acc); leaf_targets.push_back({it.b, 0}); }
    }
    for (auto& it : R) {
      if (T.bl_kind[it.b] == HM_BLOCK_SUB) subR.push_back(&it);
      else { leaf_accs.push_back(it.acc); leaf_targets.push_back({it.b, rmode}); }
    }
    // T1 of the diagonal accumulator and of the subdivided targets: one batch
    std::vector<Node*> red{&acc};
    for (auto* it : subL) red.push_back(&it->acc);
    for (auto* it : subR) red.push_back(&it->acc);
    reduce_many(red);
    std::vector<Node> ch;
    P.expand(acc, chol, ch);   // (t1,t1), (t1,t2) [chol: placeholder], (t2,t1), (t2,t2)
    const int t1 = son0(t), t2 = t1 + 1;
    std::vector<Item> L1, L2, R1, R2;
    for (auto* it : subL) {            // b = (t, r): sons (t_i, r_j), row-major
      std::vector<Node> cs;
      P.expand(it->acc, false, cs);
      const int nr = T.cl_nsons[T.bl_col[it->b]];
      for (int j = 0; j < nr; j++) {
        L1.push_back(Item{T.son(it->b, 0, j), cs[j]});
        L2.push_back(Item{T.son(it->b, 1, j), cs[nr + j]});
      }
    }
    for (auto* it : subR) {            // b = (t', t): sons (t'_i, t_j)
      std::vector<Node> cs;
      P.expand(it->acc, false, cs);
      const int nt = T.cl_nsons[T.bl_row[it->b]];
      for (int i = 0; i < nt; i++) {
        R1.push_back(Item{T.son(it->b, i, 0), cs[2 * i]});
        R2.push_back(Item{T.son(it->b, i, 1), cs[2 * i + 1]});
      }
    }
    const size_t nl = L1.size(), nr_ = R1.size();
    std::vector<Item> L1x = L1, R1x = R1;
    if (!chol) L1x.push_back(Item{blk(t1, t2), ch[1]});
    R1x.push_back(Item{blk(t2, t1), ch[2]});
    factor_merged(t1, ch[0], std::move(L1x), std::move(R1x));
    for (size_t j = 0; j < nl; j++)          // acc_(t2,r') += -L_(t2,t1) R_(t1,r')
      P.addproduct(L2[j].acc, blk(t2, t1), L1[j].b);
    for (size_t i = 0; i < nr_; i++)         // acc_(t',t2) += -L_(t',t1) R_(t1,t2)  [chol: L_(t2,t1)^T]
      P.addproduct(R2[i].acc, R1[i].b, blk(t1, t2));
    P.addproduct(ch[3], blk(t2, t1), blk(t1, t2));
    factor_merged(t2, ch[3], std::move(L2), std::move(R2));
    // leaf targets of cluster t itself: their solves run through all of L|tt / R|tt
    if (!leaf_accs.empty()) {
      flush_many(std::move(leaf_accs));
      trsm_set(t, leaf_targets);
    }
  }

  // ---- LR (O8), serial recursion (HM_FACTOR_SERIAL=1: A/B reference for factor_merged)
  void lr(int t, Node acc) {
    if (T.cl_nsons[t] == 0) {
      flush(acc);
      leaf_factor(t);
      return;
    }
    std::vector<Node> ch = split(acc, false);
    const int t1 = son0(t), t2 = t1 + 1;
    lr(t1, ch[0]);
    solve_set(t1, {Item{blk(t1, t2), ch[1]}}, {Item{blk(t2, t1), ch[2]}});
    P.addproduct(ch[3], blk(t2, t1), blk(t1, t2));
    lr(t2, ch[3]);
  }

  // ---- Cholesky (O9)
  void cholesky(int t, Node acc) {
    if (T.cl_nsons[t] == 0) {
      flush(acc);
      leaf_factor(t);
      return;
    }
    std::vector<Node> ch = split(acc, true);   // (t1,t1), [upper], (t2,t1), (t2,t2)
    const int t1 = son0(t), t2 = t1 + 1;
    cholesky(t1, ch[0]);
    solve_set(t1, {}, {Item{blk(t2, t1), ch[2]}});
    P.addproduct(ch[3], blk(t2, t1), blk(t1, t2));   // Y = L^T view: (t1,t2) of L^T = (t2,t1) of L
    cholesky(t2, ch[3]);
  }

  // compact G's admissible factors into one pool; check pivots
  void finish(double* min_pivot_out) {
    HM_CUDA(cudaStreamSynchronize(c->stream));
    int fail = 0;
    HM_CUDA(cudaMemcpy(&fail, d_fail, sizeof(int), cudaMemcpyDeviceToHost));
    std::vector<double> mp(T.nclusters());
    HM_CUDA(cudaMemcpy(mp.data(), d_minpiv, sizeof(double) * mp.size(), cudaMemcpyDeviceToHost));
    double mn = 1e300;
    for (int t = 0; t < T.nclusters(); t++)
      if (T.cl_nsons[t] == 0) mn = std::min(mn, mp[t]);
    if (min_pivot_out) *min_pivot_out = mn;
    const int nb = T.nblocks();
    size_t total = 0;
    for (int b = 0; b < nb; b++)
      if (T.bl_kind[b] == HM_BLOCK_ADM)
        total += (size_t)(T.cl_size[T.bl_row[b]] + T.cl_size[T.bl_col[b]]) * G->rank[b];
    double* pool = static_cast<double*>(c->dmalloc((total + 1) * sizeof(double)));
    size_t off = 0;
    for (int b = 0; b < nb; b++) {
      if (T.bl_kind[b] != HM_BLOCK_ADM) continue;
      const size_t m = T.cl_size[T.bl_row[b]], n = T.cl_size[T.bl_col[b]], k = G->rank[b];
      if (k) {
        HM_CUDA(cudaMemcpyAsync(pool + off, G->pA[b], sizeof(double) * m * k, cudaMemcpyDeviceToDevice, c->stream));
        HM_CUDA(cudaMemcpyAsync(pool + off + m * k, G->pB[b], sizeof(double) * n * k, cudaMemcpyDeviceToDevice,
                                c->stream));
      }
      G->pA[b] = pool + off;
      G->pB[b] = pool + off + m * k;
      off += (m + n) * k;
    }
    HM_CUDA(cudaStreamSynchronize(c->stream));
    c->dfree(G->fpool.first, G->fpool.second);
    G->fpool = {pool, (total + 1) * sizeof(double)};
    for (auto& o : own)
      if (o.first) c->dfree(o.first, o.second);
    own.clear();
    if (fail) {
      const int t = fail - 1;
      throw Error(HM_EPIVOT, "pivot breakdown in leaf cluster " + std::to_string(t) + " [" +
                                 std::to_string(T.cl_start[t]) + ":" +
                                 std::to_string(T.cl_start[t] + T.cl_size[t]) + "]");
    }
  }
};

#include "hm_std.inc"
#include "hm_solve.inc"
#include "hm_inv.inc"

}  // namespace

// Kernel-level parity export of the batched H x thin-dense product (Fig. 1
// addeval / addevaltrans) exactly as the product launches it.
void eval_batched_test(Ctx* c, Mat* H, int njobs, const int* blk, const int* trans, const double* coef,
                       const double* const* V, const int* ldv, double* const* out, const int* ldo, const int* w,
                       double split_thr) {
  const Tree& T = *H->tree;
  Planner P(c, T, H, H, H, 1.0, 0.0);
  P.setup_tables(true);
  P.split_thr = split_thr;
  Arena scratch(c);
  std::vector<EvalJob> ej;
  for (int i = 0; i < njobs; i++) {
    if (blk[i] < 0 || blk[i] >= T.nblocks()) throw Error(HM_EINVAL, "hm_test_eval_batched: bad block id");
    P.add_eval(ej, 0, blk[i], trans[i] ? 1 : 0, coef[i], out[i], ldo[i], w[i], V[i], ldv[i], 0, 0);
  }
  P.launch_evals(ej, scratch, P.fl_eval, P.by_eval);
  HM_CUDA(cudaStreamSynchronize(c->stream));
  P.persist.release();
}

// Standalone batched flush: replay the TRUNC batch of
// one captured level of the last hm_addmul from its captured stacks.
void flush_replay(Ctx* c, int level, double eps, int reps, double* ms_out, int64_t* rank_sum) {
  if (level < 0 || level >= (int)c->cap.size()) throw Error(HM_EINVAL, "hm_flush_replay: no such captured level");
  const Ctx::CapLevel& L = c->cap[level];
  if (!L.data) throw Error(HM_EINVAL, "hm_flush_replay: level captured without data (cap mask)");
  const int nj = (int)L.m.size();
  double* work = c->stack_ws(L.ndoubles + 1);
  Arena out(c);
  std::vector<double*> oa(nj), ob(nj);
  for (int i = 0; i < nj; i++) {
    const int kc = trunc_kcap(L.m[i], L.n[i], L.l[i]);
    oa[i] = out.alloc((size_t)L.m[i] * std::max(kc, 1));
    ob[i] = out.alloc((size_t)L.n[i] * std::max(kc, 1));
  }
  int* d_rank = static_cast<int*>(out.alloc_bytes(sizeof(int) * (nj + 1)));
  cudaEvent_t e0, e1;
  HM_CUDA(cudaEventCreate(&e0));
  HM_CUDA(cudaEventCreate(&e1));
  double total_ms = 0;
  std::vector<int> hr(nj);
  for (int r = 0; r < std::max(reps, 1); r++) {
    HM_CUDA(cudaMemcpyAsync(work, L.data, L.ndoubles * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
    std::vector<TruncReq> tr(nj);
    for (int i = 0; i < nj; i++)
      tr[i] = TruncReq{L.m[i], L.n[i], L.l[i], work + L.aoff[i], work + L.boff[i], oa[i], ob[i], d_rank + i, nullptr};
    Arena scratch(c);
    HM_CUDA(cudaEventRecord(e0, c->stream));
    trunc_batched(c, scratch, tr, eps);
    HM_CUDA(cudaEventRecord(e1, c->stream));
    HM_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    HM_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    total_ms += ms;
    scratch.release();
  }
  HM_CUDA(cudaMemcpy(hr.data(), d_rank, sizeof(int) * nj, cudaMemcpyDeviceToHost));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  int64_t s = 0;
  for (int i = 0; i < nj; i++) s += hr[i];
  if (rank_sum) *rank_sum = s;
  if (ms_out) *ms_out = total_ms / std::max(reps, 1);
}

void factorize(Ctx* c, Mat* G, double eps, bool chol, double shift, double* min_pivot) {
  if (!G) throw Error(HM_EINVAL, "hm_lr/hm_chol: null matrix");
  if (!(eps >= 0.0)) throw Error(HM_EINVAL, "hm_lr/hm_chol: eps must be >= 0");
  const Tree& T = *G->tree;
  if (T.bl_kind[0] != HM_BLOCK_SUB && T.bl_kind[0] != HM_BLOCK_DENSE)
    throw Error(HM_ESTRUCT, "hm_lr/hm_chol: the root block must not be admissible");
  // k_leaf_factor keeps a diagonal leaf in shared memory (m^2 doubles <= 200 KB)
  for (int t = 0; t < T.nclusters(); t++)
    if (T.cl_nsons[t] == 0 && T.cl_size[t] > kMaxLeafFactor)
      throw Error(HM_EUNSUPPORTED, "hm_lr/hm_chol: leaf cluster " + std::to_string(t) + " has " +
                                       std::to_string(T.cl_size[t]) + " rows (diagonal leaf factorization supports <= " +
                                       std::to_string(kMaxLeafFactor) + ")");
  if (shift != 0.0) {
    Arena ar(c);
    std::vector<CopyJob> cj;
    int64_t tiles = 0;
    for (int b = 0; b < T.nblocks(); b++) {
      if (T.bl_kind[b] != HM_BLOCK_DENSE || T.bl_row[b] != T.bl_col[b]) continue;
      const int m = T.cl_size[T.bl_row[b]];
      cj.push_back(CopyJob{G->pA[b], nullptr, m, 0, m, m, 0, 1, 1, shift, tiles});
      tiles += (int64_t)((m + 31) / 32) * ((m + 31) / 32);
    }
    launch_copy_mapped(ar.upload(cj), (int)cj.size(), ar.tile_map(cj, tiles), tiles, c->stream);
    HM_CHECK_LAUNCH();
  }
  c->sp_prepare();
  Factorizer F(c, G, eps, chol);
  Node root = F.acc_for(0);
  const int t = T.bl_row[0];
  static const bool serial = std::getenv("HM_FACTOR_SERIAL") != nullptr;
  if (!serial) F.factor_merged(t, root, {}, {});
  else if (chol) F.cholesky(t, root);
  else F.lr(t, root);
  F.finish(min_pivot);
  if (std::getenv("HM_DEBUG_TIMING"))
    std::fprintf(stderr,
                 "[hm_factor] flushes %lld (calls %lld, reduce calls %lld) trsm %lld leaf %lld syncs %lld | planner: levels %.3fs (sync wait %.3fs; host "
                 "layout %.3f jobs %.3f launch %.3f trunc %.3f) split %.3fs merges %.3fs\n",
                 (long long)F.n_flush, (long long)F.n_flush_calls, (long long)F.n_reduce_calls, (long long)F.n_trsm, (long long)F.n_leaf, (long long)F.P.n_sync, F.P.t_level, F.P.t_wait,
                 F.P.t_a, F.P.t_b, F.P.t_c, F.P.t_d, F.P.t_split, F.P.t_merge);
  hm_stats_t& s = c->last;
  s.addproduct_calls = F.P.n_addproduct;
  s.evaluated_terms = F.P.n_eval;
  s.truncations = F.P.n_trunc;
  s.trunc_cols = F.P.n_cols;
  s.merges = F.P.n_merge;
  s.dense_adds = F.P.n_dense;
  s.levels = F.n_flush;
  s.flops_trunc = F.P.fl_trunc;
  s.bytes_trunc = F.P.by_trunc;
  s.flops_eval = F.P.fl_eval;
  s.bytes_eval = F.P.by_eval;
  s.flops_dense = F.P.fl_dense;
  s.bytes_dense = F.P.by_dense;
  F.P.persist.release();
  HM_CUDA(cudaStreamSynchronize(c->stream));
}

void solve_thin(Ctx* c, Mat* F, int part, double* x, int64_t ldx, int ncols) {
  if (!F || !x || ncols < 0 || ldx < F->tree->n) throw Error(HM_EINVAL, "hm_solve_thin: bad arguments");
  if (part < 0 || part > 5) throw Error(HM_EINVAL, "hm_solve_thin: unknown operator");
  Solver S(c, F, part);
  S.run(x, (int)ldx, ncols);
}

// ||I - F^{-1} G0||_2 by power iteration on E^T E (oracle
// factor.precond_error): F = L R (kind 0) or L L^T (kind 1) in place.
double precond_error(Ctx* c, Mat* G0, Mat* F, int kind, int iters, uint64_t seed) {
  if (!G0 || !F || iters <= 0 || kind < 0 || kind > 2) throw Error(HM_EINVAL, "hm_precond_error: bad arguments");
  if (!G0->tree->same_structure(*F->tree)) throw Error(HM_ESTRUCT, "hm_precond_error: G and F trees differ");
  const int64_t n = F->tree->n;
  cudaStream_t st = c->stream;
  Arena ar(c);
  double* v = ar.alloc(n);
  double* y = ar.alloc(n);
  double* w = ar.alloc(n);
  double* d_nrm = ar.alloc(8);
  const NormJob* dj_v = ar.upload(std::vector<NormJob>{NormJob{v, (int)n, 1, (int)n, nullptr}});
  const NormJob* dj_w = ar.upload(std::vector<NormJob>{NormJob{w, (int)n, 1, (int)n, nullptr}});
  auto norm = [&](const NormJob* j) {
    launch_norm(j, 1, d_nrm, st);
    double h = 0;
    HM_CUDA(cudaMemcpyAsync(&h, d_nrm, sizeof(double), cudaMemcpyDeviceToHost, st));
    HM_CUDA(cudaStreamSynchronize(st));
    return std::sqrt(h);
  };
  // kind 0 / 1: F^{-1} by the factor solves; kind 2: F = the inverse itself (hm_inv)
  std::unique_ptr<Solver> s1, s2, t1, t2;
  if (kind != 2) {
    s1.reset(new Solver(c, F, kind == 0 ? 0 : 4));
    s2.reset(new Solver(c, F, kind == 0 ? 1 : 5));
  }
  if (kind == 0) {   // F^{-T} = L^{-T} R^{-T}
    t1.reset(new Solver(c, F, 3));
    t2.reset(new Solver(c, F, 2));
  }
  double* tmp = kind == 2 ? ar.alloc(n) : nullptr;
  launch_randn(v, n, seed, st);
  double nv = norm(dj_v);
  launch_axpby(0.0, v, n, 1.0 / nv, v, n, n, 1, st);
  double est = 0;
  for (int it = 0; it < iters; it++) {
    if (kind == 2) {
      matvec(c, G0, HM_OP_G, 1.0, v, n, 0.0, tmp, n, 1);         // y = Ginv (G v)
      matvec(c, F, HM_OP_G, 1.0, tmp, n, 0.0, y, n, 1);
    } else {
      matvec(c, G0, HM_OP_G, 1.0, v, n, 0.0, y, n, 1);            // y = G v
      s1->rec(F->tree->bl_row[0], y, (int)n, 1);                    // y = F^{-1} G v
      s2->rec(F->tree->bl_row[0], y, (int)n, 1);
    }
    launch_axpby(1.0, v, n, 0.0, w, n, n, 1, st);                  // w = v - y = E v
    launch_axpby(-1.0, y, n, 1.0, w, n, n, 1, st);
    est = norm(dj_w);
    if (est == 0.0) break;
    launch_axpby(1.0, w, n, 0.0, y, n, n, 1, st);                  // y = F^{-T} w
    if (kind == 0) {
      t1->rec(F->tree->bl_row[0], y, (int)n, 1);
      t2->rec(F->tree->bl_row[0], y, (int)n, 1);
    } else if (kind == 1) {
      s1->rec(F->tree->bl_row[0], y, (int)n, 1);
      s2->rec(F->tree->bl_row[0], y, (int)n, 1);
    } else {
      matvec(c, F, HM_OP_GT, 1.0, w, n, 0.0, y, n, 1);            // y = Ginv^T w
    }
    matvec(c, G0, HM_OP_GT, 1.0, y, n, 0.0, v, n, 1);             // v = G^T F^{-T} w
    launch_axpby(1.0, w, n, -1.0, v, n, n, 1, st);                 // v = w - v = E^T E v_old
    nv = norm(dj_v);
    if (nv == 0.0) break;
    launch_axpby(0.0, v, n, 1.0 / nv, v, n, n, 1, st);
  }
  HM_CUDA(cudaStreamSynchronize(st));
  return est;
}

// H-inversion with accumulated updates (Fig. 8): G <- approximate G^{-1}
void invert_matrix(Ctx* c, Mat* G, double eps, double* min_pivot) {
  if (!G) throw Error(HM_EINVAL, "hm_inv: null matrix");
  if (!(eps >= 0.0)) throw Error(HM_EINVAL, "hm_inv: eps must be >= 0");
  const Tree& T = *G->tree;
  if (T.bl_kind[0] == HM_BLOCK_ADM) throw Error(HM_ESTRUCT, "hm_inv: the root block must not be admissible");
  for (int t = 0; t < T.nclusters(); t++)
    if (T.cl_nsons[t] == 0 && T.cl_size[t] > kMaxLeafFactor)
      throw Error(HM_EUNSUPPORTED, "hm_inv: leaf cluster larger than " + std::to_string(kMaxLeafFactor) + " rows");
  const int nb = T.nblocks();
  Mat H;   // auxiliary H-matrix: same tree, zero
  H.tree = G->tree;
  H.rank.assign(nb, 0);
  H.pA.assign(nb, nullptr);
  H.pB.assign(nb, nullptr);
  size_t nd = 0;
  for (int b = 0; b < nb; b++)
    if (T.bl_kind[b] == HM_BLOCK_DENSE) nd += (size_t)T.cl_size[T.bl_row[b]] * T.cl_size[T.bl_col[b]];
  double* dp = static_cast<double*>(c->dmalloc((nd + 1) * sizeof(double)));
  H.dpool = {dp, (nd + 1) * sizeof(double)};
  HM_CUDA(cudaMemsetAsync(dp, 0, (nd + 1) * sizeof(double), c->stream));
  size_t off = 0;
  for (int b = 0; b < nb; b++)
    if (T.bl_kind[b] == HM_BLOCK_DENSE) {
      H.pA[b] = dp + off;
      off += (size_t)T.cl_size[T.bl_row[b]] * T.cl_size[T.bl_col[b]];
    }
  c->sp_prepare();
  {
    Inverter I(c, G, &H, eps);
    I.invert(T.bl_row[0], I.acc_for(0, 0));
    I.finish(min_pivot);
    hm_stats_t& s = c->last;
    s.addproduct_calls = I.P.n_addproduct;
    s.evaluated_terms = I.P.n_eval;
    s.truncations = I.P.n_trunc;
    s.trunc_cols = I.P.n_cols;
    s.merges = I.P.n_merge;
    s.dense_adds = I.P.n_dense;
    s.levels = I.n_flush;
    s.flops_trunc = I.P.fl_trunc;
    s.bytes_trunc = I.P.by_trunc;
    s.flops_eval = I.P.fl_eval;
    s.bytes_eval = I.P.by_eval;
    s.flops_dense = I.P.fl_dense;
    s.bytes_dense = I.P.by_dense;
    I.P.persist.release();
  }
  H.free_all(c);
  HM_CUDA(cudaStreamSynchronize(c->stream));
}

void addmul_std(Ctx* c, double alpha, Mat* X, Mat* Y, Mat* Z, double eps) {
  if (!X || !Y || !Z) throw Error(HM_EINVAL, "hm_addmul_std: null matrix");
  if (Z == X || Z == Y) throw Error(HM_ESTRUCT, "hm_addmul_std: Z aliases X or Y (use hm_clone)");
  if (!(eps >= 0.0)) throw Error(HM_EINVAL, "hm_addmul_std: eps must be >= 0");
  const Tree& T = *Z->tree;
  if (!(X->tree->same_structure(T) && Y->tree->same_structure(T)))
    throw Error(HM_ESTRUCT, "hm_addmul_std: X, Y and Z must share one block tree");
  c->sp_prepare();
  StdExec S(c, X, Y, Z, alpha, eps);
  S.run(Z);
  hm_stats_t& s = c->last;
  s = hm_stats_t{};
  s.addproduct_calls = S.n_addproduct;
  s.evaluated_terms = (int64_t)S.terms.size();
  s.truncations = S.P.n_trunc;
  s.trunc_cols = S.P.n_cols;
  s.merges = S.n_m;
  s.dense_adds = S.P.n_dense;
  s.levels = S.rounds;
  s.flops_trunc = S.P.fl_trunc;
  s.bytes_trunc = S.P.by_trunc;
  s.flops_eval = S.P.fl_eval;
  s.bytes_eval = S.P.by_eval;
  s.flops_dense = S.P.fl_dense;
  s.bytes_dense = S.P.by_dense;
  S.P.persist.release();
  HM_CUDA(cudaStreamSynchronize(c->stream));
}

void addmul(Ctx* c, double alpha, Mat* X, Mat* Y, Mat* Z, double eps) {
  if (!X || !Y || !Z) throw Error(HM_EINVAL, "hm_addmul: null matrix");
  if (Z == X || Z == Y) throw Error(HM_ESTRUCT, "hm_addmul: Z aliases X or Y (use hm_clone)");
  if (!(eps >= 0.0)) throw Error(HM_EINVAL, "hm_addmul: eps must be >= 0");
  const Tree& T = *Z->tree;
  if (!(X->tree->same_structure(T) && Y->tree->same_structure(T)))
    throw Error(HM_ESTRUCT, "hm_addmul: X, Y and Z must share one block tree");
  c->sp_prepare();
  Planner P(c, T, X, Y, Z, alpha, eps);
  if (c->cap_on) {
    c->cap_free();
    P.capture = true;
  }
  P.run();
  c->cap_on = false;
  hm_stats_t& s = c->last;
  s.addproduct_calls = P.n_addproduct;
  s.evaluated_terms = P.n_eval;
  s.truncations = P.n_trunc;
  s.trunc_cols = P.n_cols;
  s.merges = P.n_merge;
  s.dense_adds = P.n_dense;
  s.levels = (int64_t)P.levels.size();
  s.flops_trunc = P.fl_trunc;
  s.bytes_trunc = P.by_trunc;
  s.flops_eval = P.fl_eval;
  s.bytes_eval = P.by_eval;
  s.flops_dense = P.fl_dense;
  s.bytes_dense = P.by_dense;
  P.persist.release();
  HM_CUDA(cudaStreamSynchronize(c->stream));
}

}  // namespace hm
