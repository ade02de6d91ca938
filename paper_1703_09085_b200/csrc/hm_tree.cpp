// Cluster tree and block tree (PAPER.md Defs 2.1-2.2) built on the
// host with the rules of DESIGN.md §4 (bounding-box bisection at the
// midpoint of the longest axis; admissibility max(d_t^2, d_s^2) <= eta^2 dist^2).
// Compiled with -ffp-contract=off so every comparison is evaluated in the
// same FP64 operation order as the specification.
#include <algorithm>
#include <cmath>
#include <deque>
#include <functional>

#include "hm_internal.h"

namespace hm {

namespace {
struct TmpCluster {
  int start, size, level;
  double lo[3], hi[3];
  int son[2] = {-1, -1};
  int nsons = 0;
};

void bbox(const double* pts, const int64_t* idx, int cnt, double* lo, double* hi) {
  for (int a = 0; a < 3; a++) {
    double l = pts[3 * idx[0] + a], h = l;
    for (int i = 1; i < cnt; i++) {
      const double v = pts[3 * idx[i] + a];
      if (v < l) l = v;
      if (v > h) h = v;
    }
    lo[a] = l;
    hi[a] = h;
  }
}

double diam2(const double* lo, const double* hi) {
  double d = 0.0;
  for (int a = 0; a < 3; a++) {
    const double e = hi[a] - lo[a];
    d = d + e * e;
  }
  return d;
}

double dist2(const double* tl, const double* th, const double* sl, const double* sh) {
  double d = 0.0;
  for (int a = 0; a < 3; a++) {
    double g = sl[a] - th[a];
    const double g2 = tl[a] - sh[a];
    if (g2 > g) g = g2;
    if (0.0 > g) g = 0.0;
    d = d + g * g;
  }
  return d;
}
}  // namespace

std::shared_ptr<Tree> build_trees(const double* pts, int64_t n, int leaf_size, double eta) {
  if (n <= 0) throw Error(HM_EINVAL, "hm_build: n must be positive");
  if (leaf_size < 1) throw Error(HM_EINVAL, "hm_build: leaf_size must be >= 1");
  if (!(eta > 0.0)) throw Error(HM_EINVAL, "hm_build: eta must be positive");
  auto T = std::make_shared<Tree>();
  T->n = n;
  T->perm.resize(n);
  for (int64_t i = 0; i < n; i++) T->perm[i] = i;
  std::vector<TmpCluster> cl;
  cl.reserve(4 * (n / leaf_size + 1));
  TmpCluster root{};
  root.start = 0;
  root.size = (int)n;
  root.level = 0;
  bbox(pts, T->perm.data(), (int)n, root.lo, root.hi);
  cl.push_back(root);
  std::vector<int> stack{0};
  std::vector<int64_t> left, right;
  while (!stack.empty()) {
    const int ci = stack.back();
    stack.pop_back();
    TmpCluster c = cl[ci];
    if (c.size <= leaf_size) continue;
    int64_t* idx = T->perm.data() + c.start;
    int ax = 0;
    double ext[3];
    for (int a = 0; a < 3; a++) ext[a] = c.hi[a] - c.lo[a];
    for (int a = 1; a < 3; a++)
      if (ext[a] > ext[ax]) ax = a;
    const double mid = 0.5 * (c.lo[ax] + c.hi[ax]);
    left.clear();
    right.clear();
    for (int i = 0; i < c.size; i++) {
      if (pts[3 * idx[i] + ax] < mid) left.push_back(idx[i]); else right.push_back(idx[i]);
    }
    if (left.empty() || right.empty()) {
      std::vector<int64_t> all(idx, idx + c.size);
      left.assign(all.begin(), all.begin() + c.size / 2);
      right.assign(all.begin() + c.size / 2, all.end());
    }
    std::copy(left.begin(), left.end(), idx);
    std::copy(right.begin(), right.end(), idx + left.size());
    const int nl = (int)left.size();
    for (int s = 0; s < 2; s++) {
      TmpCluster sc{};
      sc.start = c.start + (s == 0 ? 0 : nl);
      sc.size = (s == 0) ? nl : c.size - nl;
      sc.level = c.level + 1;
      bbox(pts, T->perm.data() + sc.start, sc.size, sc.lo, sc.hi);
      cl.push_back(sc);
      cl[ci].son[s] = (int)cl.size() - 1;
    }
    cl[ci].nsons = 2;
    stack.push_back(cl[ci].son[0]);
    stack.push_back(cl[ci].son[1]);
  }
  // breadth-first numbering
  std::vector<int> bfs;
  bfs.reserve(cl.size());
  std::vector<int> newid(cl.size(), -1);
  std::deque<int> q{0};
  while (!q.empty()) {
    const int c = q.front();
    q.pop_front();
    newid[c] = (int)bfs.size();
    bfs.push_back(c);
    for (int s = 0; s < cl[c].nsons; s++) q.push_back(cl[c].son[s]);
  }
  const int nc = (int)bfs.size();
  T->cl_start.resize(nc);
  T->cl_size.resize(nc);
  T->cl_son0.resize(nc);
  T->cl_nsons.resize(nc);
  T->cl_level.resize(nc);
  T->cl_bbox.resize(6 * (size_t)nc);
  for (int i = 0; i < nc; i++) {
    const TmpCluster& c = cl[bfs[i]];
    T->cl_start[i] = c.start;
    T->cl_size[i] = c.size;
    T->cl_nsons[i] = c.nsons;
    T->cl_son0[i] = c.nsons ? newid[c.son[0]] : -1;
    T->cl_level[i] = c.level;
    for (int a = 0; a < 3; a++) {
      T->cl_bbox[6 * i + a] = c.lo[a];
      T->cl_bbox[6 * i + 3 + a] = c.hi[a];
    }
  }
  // block tree, breadth first
  const double eta2 = eta * eta;
  std::deque<std::pair<int, int>> bq{{0, 0}};
  std::vector<int> parent_son0;  // not needed; sons are appended consecutively
  while (!bq.empty()) {
    auto [t, s] = bq.front();
    bq.pop_front();
    const int id = (int)T->bl_row.size();
    T->bl_row.push_back(t);
    T->bl_col.push_back(s);
    T->bl_level.push_back(T->cl_level[t]);
    const double* tl = &T->cl_bbox[6 * t];
    const double* th = tl + 3;
    const double* sl = &T->cl_bbox[6 * s];
    const double* sh = sl + 3;
    const double dt = diam2(tl, th), ds = diam2(sl, sh);
    const double dmax = dt > ds ? dt : ds;
    int kind;
    if (dmax <= eta2 * dist2(tl, th, sl, sh)) kind = HM_BLOCK_ADM;
    else if (T->cl_nsons[t] == 0 || T->cl_nsons[s] == 0) kind = HM_BLOCK_DENSE;
    else kind = HM_BLOCK_SUB;
    T->bl_kind.push_back(kind);
    T->bl_son0.push_back(-1);
    T->bl_nsons.push_back(0);
    if (kind == HM_BLOCK_SUB) {
      // sons get ids in BFS order: current queue length + already numbered
      T->bl_son0[id] = id + 1 + (int)bq.size();
      T->bl_nsons[id] = T->cl_nsons[t] * T->cl_nsons[s];
      for (int i = 0; i < T->cl_nsons[t]; i++)
        for (int j = 0; j < T->cl_nsons[s]; j++)
          bq.push_back({T->cl_son0[t] + i, T->cl_son0[s] + j});
    }
  }
  T->finalize();
  return T;
}

void Tree::finalize() {
  const int nb = nblocks();
  bl_lbeg.assign(nb, 0);
  bl_lend.assign(nb, 0);
  leaf_order.clear();
  if (bl_level.size() != (size_t)nb) {
    bl_level.resize(nb);
    for (int b = 0; b < nb; b++) bl_level[b] = cl_level[bl_row[b]];
  }
  depth = 0;
  for (int b = 0; b < nb; b++) depth = std::max(depth, bl_level[b]);
  // iterative DFS computing leaf ranges
  std::vector<std::pair<int, int>> st{{0, 0}};
  while (!st.empty()) {
    auto& [b, state] = st.back();
    if (state == 0) {
      bl_lbeg[b] = (int)leaf_order.size();
      if (bl_kind[b] != HM_BLOCK_SUB) {
        leaf_order.push_back(b);
        bl_lend[b] = (int)leaf_order.size();
        st.pop_back();
        continue;
      }
      state = 1;
      const int b0 = bl_son0[b], ns = bl_nsons[b];
      for (int i = ns - 1; i >= 0; i--) st.push_back({b0 + i, 0});
    } else {
      bl_lend[b] = (int)leaf_order.size();
      st.pop_back();
    }
  }
}

bool Tree::same_structure(const Tree& o) const {
  return n == o.n && cl_start == o.cl_start && cl_size == o.cl_size && cl_son0 == o.cl_son0 &&
         cl_nsons == o.cl_nsons && bl_row == o.bl_row && bl_col == o.bl_col && bl_kind == o.bl_kind &&
         bl_son0 == o.bl_son0 && bl_nsons == o.bl_nsons;
}

}  // namespace hm
