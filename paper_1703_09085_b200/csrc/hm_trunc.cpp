// Batched TRUNC_eps (§3 "Truncation" P:L336-384, Fig. 2 rkadd
// P:L416-436): for every stack (A, B) compute the eps-truncated SVD of the
// exact A B^T.
//
// Route on the device: Householder QR of A if l < m and of B
// if l < n (otherwise that factor is used as is), M = R_A R_B^T (p x q), one-sided
// Jacobi SVD of M with the relative-Frobenius rank rule, then
// A' = Q_A [U_k; 0], B' = Q_B [V_k S_k; 0].  Same exact matrix as the oracle's
// route (QR of B, SVD of A R_B^T), so ranks and represented matrices agree up
// to rounding.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "hm_internal.h"

namespace hm {

int trunc_kcap(int m, int n, int l) {
  const int p = l < m ? l : m;
  const int q = l < n ? l : n;
  return std::min(p, q);
}

double trunc_flops(double m, double n, double l, double k) {
  // QR path 2(m+n)l^2 - 4/3 l^3 + l^3/3 + 22 l^3 + 2(m+n) l k ;
  // dense path (l >= min(m,n)): 2 m n l + 14 p q^2 + 8 q^3.
  if (l <= 0) return 0.0;
  if (l < std::min(m, n))
    return 2.0 * (m + n) * l * l - (4.0 / 3.0) * l * l * l + l * l * l / 3.0 + 22.0 * l * l * l +
           2.0 * (m + n) * l * k;
  const double p = std::max(m, n), q = std::min(m, n);
  return 2.0 * m * n * l + 14.0 * p * q * q + 8.0 * q * q * q;
}

double trunc_bytes(double m, double n, double l, double k) {
  return 8.0 * (m + n) * (l + k);
}

namespace {
int bucket_cap(int64_t need) {
  if (need <= 3 * 1024) return 3 * 1024;
  if (need <= 8 * 1024) return 8 * 1024;
  if (need <= 26 * 1024) return 26 * 1024;
  return 0;  // global path
}
}  // namespace

static void trunc_general(Ctx* c, Arena& ar, const std::vector<TruncReq>& reqs, double eps);

// Stacks whose whole working set fits in shared memory go to the fused
// single-kernel TRUNC (k_trunc_small); the others to the staged pipeline.
void trunc_batched(Ctx* c, Arena& ar, const std::vector<TruncReq>& reqs, double eps) {
  if (reqs.empty()) return;
  if (const char* dump = std::getenv("HM_DUMP_TRUNC")) {   // diagnostics: shapes of every batch
    if (FILE* f = std::fopen(dump, "a")) {
      for (const TruncReq& r : reqs) std::fprintf(f, "%d %d %d\n", r.m, r.n, r.l);
      std::fprintf(f, "#\n");
      std::fclose(f);
    }
  }
  // (13 K doubles = 104 KB: the largest working set of which two CTAs share an SM)
  constexpr int kFB = 4;
  std::vector<TruncSmallJob> fb[kFB];
  const int fcap[kFB] = {4 * 1024, 10 * 1024, 13 * 1024, 26 * 1024};
  std::vector<TruncReq> rest;
  static const bool no_fused = std::getenv("HM_NO_FUSED") != nullptr;
  double fl = 0, by = 0;
  for (const TruncReq& r : reqs) {
    const int need = trunc_small_need(r.m, r.n, r.l);
    int b = -1;
    for (int k = 0; k < kFB; k++)
      if (need <= fcap[k]) { b = k; break; }
    if (b < 0 || no_fused) { rest.push_back(r); continue; }
    fb[b].push_back(TruncSmallJob{r.A, r.B, r.m, r.n, r.l, r.Aout, r.Bout, r.d_rank, r.d_sigma});
    fl += trunc_flops(r.m, r.n, r.l, 0.0);   // convention flops (reform term k unknown here)
    by += trunc_bytes(r.m, r.n, r.l, 0.0);
  }
  // few stacks (latency-bound steps): the 13 K and 26 K buckets share one launch
  if (!fb[2].empty() && fb[2].size() + fb[3].size() < 296) {
    fb[3].insert(fb[3].end(), fb[2].begin(), fb[2].end());
    fb[2].clear();
  }
  if (c->plog) {
    int mx = 0, ml = 0, nf = 0;
    for (int b = 0; b < kFB; b++)
      for (auto& j : fb[b]) { mx = std::max(mx, std::max(j.m, j.n)); ml = std::max(ml, j.l); nf++; }
    c->prof_note("fused jobs " + std::to_string(nf) + " maxmn " + std::to_string(mx) + " maxl " + std::to_string(ml) +
                 " staged " + std::to_string(rest.size()));
  }
  // the fused small stacks and the staged pipeline of the larger ones are
  // independent: the fused kernels run on an auxiliary stream next to it
  bool forked = false;
  {
    const TruncSmallJob* dj[kFB];
    bool any = false;
    for (int b = 0; b < kFB; b++) {
      dj[b] = fb[b].empty() ? nullptr : ar.upload_t(fb[b]);
      any = any || dj[b];
    }
    if (any) {
      forked = !rest.empty() && c->multi_stream();
      cudaStream_t sf = forked ? c->fork(0) : c->stream;
      ProfScope ps(c, PC_FUSED, fl, by, sf);
      for (int b = 0; b < kFB; b++)
        if (dj[b]) launch_trunc_small(dj[b], (int)fb[b].size(), eps, fcap[b], sf);
      HM_CHECK_LAUNCH();
    }
  }
  trunc_general(c, ar, rest, eps);
  if (forked) c->join(0);
}

static void trunc_general(Ctx* c, Arena& ar, const std::vector<TruncReq>& reqs, double eps) {
  if (reqs.empty()) return;
  cudaStream_t st = c->stream;
  const int nj = (int)reqs.size();
  std::string shapes;
  if (c->plog) {
    for (int i = 0; i < nj && i < 6; i++)
      shapes += " " + std::to_string(reqs[i].m) + "x" + std::to_string(reqs[i].n) + "x" + std::to_string(reqs[i].l);
    shapes = "jobs " + std::to_string(nj) + shapes;
  }
  std::vector<int> p(nj), q(nj);
  std::vector<char> qa(nj), qb(nj);
  size_t tau_total = 0, m_total = 0;
  for (int i = 0; i < nj; i++) {
    const TruncReq& r = reqs[i];
    // one-sided route (the paper's: QR of one factor, SVD of A R_B^*): QR the
    // factor with more rows if the stack is thin there; the column-pivoted QR
    // inside the SVD kernel orthogonalises the other side.
    if (r.n >= r.m) { qa[i] = 0; qb[i] = r.l < r.n; }
    else { qa[i] = r.l < r.m; qb[i] = 0; }
    // both factors tall and the one-sided M (min(m,n) x l) too large for shared
    // memory: QR both (two independent CTAs) so M = R_A R_B^T is only l x l --
    // avoids a third, sequential QR of M on the critical path
    static const int64_t both_thr = [] { const char* e = std::getenv("HM_QR_BOTH_THR"); return e ? std::atoll(e) : (int64_t)12 * 1024; }();
    if (r.l < r.m && r.l < r.n && (int64_t)std::min(r.m, r.n) * r.l > both_thr) qa[i] = qb[i] = 1;
    p[i] = qa[i] ? r.l : r.m;
    q[i] = qb[i] ? r.l : r.n;
    if (qa[i]) tau_total += r.l;
    if (qb[i]) tau_total += r.l;
    m_total += (size_t)p[i] * q[i];
  }
  double* tau = ar.alloc(tau_total + 1);
  double* Mbuf = ar.alloc(m_total + 1);
  // --- tall thin factors get a TSQR plan: the factor is cut into chunks of h
  // rows, every chunk is QR'd by its own CTA, the chunk R's are stacked
  // (upper triangles, zeros below) and the stack is QR'd the same way until one
  // chunk remains.  Same factorisation A = Q R (Q = blockdiag(Q_chunks) Q_stack,
  // R = the last level's R), but the single-CTA row sweep over thousands of
  // rows becomes nch independent CTAs.
  static const int ts_min_b = [] { const char* e = std::getenv("HM_TSQR_ROWS"); return e ? std::atoi(e) : 768; }();
  static const int ts_h_b = [] { const char* e = std::getenv("HM_TSQR_H"); return e ? std::atoi(e) : 768; }();
  // small batches (latency-bound, e.g. the H-LR critical path) may cut tall
  // factors into more, shorter chunks (more CTAs on one QR)
  static const int ts_min_l = [] { const char* e = std::getenv("HM_TSQR_ROWS_LAT"); return e ? std::atoi(e) : 768; }();
  static const int ts_h_l = [] { const char* e = std::getenv("HM_TSQR_H_LAT"); return e ? std::atoi(e) : 768; }();
  static const int ts_even = [] { const char* e = std::getenv("HM_TSQR_EVEN"); return e ? std::atoi(e) : 1; }();
  const bool lat_batch = nj < 64;
  const int ts_min = lat_batch ? ts_min_l : ts_min_b;
  const int ts_h = lat_batch ? ts_h_l : ts_h_b;
  struct TsLevel { double* V; int rows, ld, h, nch; double* tau; size_t xoff; double* X; int ldx; double* T; };
  struct TsPlan { int job, side, l, kcap; std::vector<TsLevel> lv; };
  std::vector<TsPlan> ts;
  std::vector<int> tsp[2] = {std::vector<int>(nj, -1), std::vector<int>(nj, -1)};
  size_t xslab = 0;
  for (int i = 0; i < nj; i++) {
    const TruncReq& r = reqs[i];
    for (int side = 0; side < 2; side++) {
      const int rows0 = side == 0 ? r.m : r.n;
      if (!(side == 0 ? qa[i] : qb[i]) || ts_min <= 0 || rows0 <= ts_min || 2 * r.l > ts_h) continue;
      TsPlan P{i, side, r.l, trunc_kcap(r.m, r.n, r.l), {}};
      TsLevel L{side == 0 ? r.A : r.B, rows0, rows0, 0, 1, nullptr, 0, side == 0 ? r.Aout : r.Bout, rows0, nullptr};
      for (;;) {
        if (L.rows > ts_min) {
          if (ts_even) {   // chunks of equal height <= ts_h (every chunk in the register-panel QR's range)
            L.nch = (L.rows + ts_h - 1) / ts_h;
            L.h = (L.rows + L.nch - 1) / L.nch;
          } else {         // chunks of ts_h rows, the last one takes the remainder (< 2 ts_h)
            L.h = ts_h;
            L.nch = L.rows / ts_h;
          }
        } else { L.h = L.rows; L.nch = 1; }
        L.tau = ar.alloc((size_t)L.nch * r.l);
        L.T = ar.alloc((size_t)L.nch * ((r.l + 15) / 16) * 256);
        P.lv.push_back(L);
        if (L.nch == 1) break;
        const int rows = L.nch * r.l;
        L = TsLevel{ar.alloc((size_t)rows * r.l), rows, rows, 0, 1, nullptr, xslab, nullptr, rows, nullptr};
        xslab += (size_t)rows * P.kcap;
      }
      tsp[side][i] = (int)ts.size();
      ts.push_back(std::move(P));
    }
  }
  double* xbuf = xslab ? ar.alloc(xslab) : nullptr;
  size_t maxdepth = 0;
  for (TsPlan& P : ts) {
    for (size_t j = 1; j < P.lv.size(); j++) P.lv[j].X = xbuf + P.lv[j].xoff;
    maxdepth = std::max(maxdepth, P.lv.size());
  }
  auto chunk = [](const TsLevel& L, int ch, int& r0, int& rows) {
    r0 = ch * L.h;
    rows = ch == L.nch - 1 ? L.rows - r0 : L.h;
  };
  auto chunkT = [](const TsLevel& L, int ch, int rows, int l) -> double* {
    return qr_has_T(rows, l) ? L.T + (size_t)ch * ((l + 15) / 16) * 256 : nullptr;
  };
  // --- QR jobs, bucketed by shared-memory need
  static const int qr_stepped = [] { const char* e = std::getenv("HM_QR_STEPPED"); return e ? std::atoi(e) : 1; }();
  static const int qr_stepped_min = [] { const char* e = std::getenv("HM_QR_STEPPED_MIN"); return e ? std::atoi(e) : 32; }();
  auto stepped_ok = [&](int njobs) { return qr_stepped && njobs >= qr_stepped_min; };
  // bucket b <= 2 (m <= 1536, every job has a T buffer): stepped QR for batches,
  // the one-CTA-per-job kernel for the few-job (latency-bound) case
  // buckets 0 / 1 (m <= 768): register-panel QR (qr_reg.cu), one launch per row
  // class (the class fixes threads and rows per thread); HM_QR_REG=0: the
  // shared-memory-panel kernels
  static const int qr_reg = [] { const char* e = std::getenv("HM_QR_REG"); return e ? std::atoi(e) : 1; }();
  auto qr_class = [](int m) { return m <= 128 ? 0 : (m <= 256 ? 1 : (m <= 384 ? 2 : (m <= 512 ? 3 : 4))); };
  // order of a bucket's jobs before the upload
  auto prep_bucket = [&](std::vector<QrJob>& v, int b) {
    if (b <= 1 && qr_reg)
      std::stable_sort(v.begin(), v.end(), [&](const QrJob& x, const QrJob& y) { return qr_class(x.m) < qr_class(y.m); });
    else if (b <= 2 && stepped_ok((int)v.size()))
      std::stable_sort(v.begin(), v.end(), [](const QrJob& x, const QrJob& y) { return x.n > y.n; });
  };
  auto launch_bucket = [&](const std::vector<QrJob>& v, const QrJob* dv, int b, int cap, cudaStream_t s) {
    if (b <= 1 && qr_reg) {
      for (size_t i0 = 0; i0 < v.size();) {
        const int cl = qr_class(v[i0].m);
        size_t i1 = i0;
        int mm = 0;
        while (i1 < v.size() && qr_class(v[i1].m) == cl) { mm = std::max(mm, v[i1].m); i1++; }
        launch_qr_reg(dv + i0, (int)(i1 - i0), mm, s);
        i0 = i1;
      }
    } else if (b <= 2 && stepped_ok((int)v.size())) {
      std::vector<int> nc(v.size());
      int mm = 0;
      for (size_t i = 0; i < v.size(); i++) { nc[i] = v[i].n; mm = std::max(mm, v[i].m); }
      launch_qr_stepped(dv, nc.data(), (int)v.size(), mm, s);
    } else {
      launch_qr_blocked(dv, (int)v.size(), cap, s);
    }
  };
  auto launch_qr_set = [&](const std::vector<QrJob>& jobs) {
    std::vector<QrJob> qs, qbk[4], qr_huge;
    for (const QrJob& j : jobs) {
      const int64_t need = (int64_t)j.m * j.n;
      if (need <= 4 * 1024) { qs.push_back(j); continue; }
      if (j.m > 24 * 1024) { qr_huge.push_back(j); continue; }
      const int b = j.m <= 384 ? 0 : (j.m <= 768 ? 1 : (j.m <= 1536 ? 2 : 3));
      qbk[b].push_back(j);
    }
    // stepped QR (qr.cu): jobs sorted by column count, so that every panel step
    // launches only the prefix of jobs that still has columns left
    for (int b = 0; b < 3; b++) prep_bucket(qbk[b], b);
    // uploads first (they are ordered on the main stream), then every bucket
    // on its own auxiliary stream: the buckets are independent problems
    const QrJob* dqs = qs.empty() ? nullptr : ar.upload_t(qs);
    const QrJob* dqh = qr_huge.empty() ? nullptr : ar.upload_t(qr_huge);
    const QrJob* dqb[4];
    int used = (dqs ? 1 : 0) + (dqh ? 1 : 0);
    for (int b = 0; b < 4; b++) {
      dqb[b] = qbk[b].empty() ? nullptr : ar.upload_t(qbk[b]);
      used += dqb[b] ? 1 : 0;
    }
    const bool par = used > 1 && c->multi_stream();
    // blocked (compact-WY) QR, bucketed by panel height so that small panels
    // get several CTAs per SM: cap = 16 * rows doubles of shared memory
    const int qcap[4] = {6 * 1024, 12 * 1024, 24 * 1024, 24 * 1024};
    for (int b = 3; b >= 0; b--)
      if (dqb[b]) {
        cudaStream_t sb = par ? c->fork(1 + b) : st;
        ProfScope pb(c, PC_QR_B0 + b, 0, (double)qbk[b].size(), sb);
        launch_bucket(qbk[b], dqb[b], b, qcap[b], sb);
      }
    if (dqs) {
      ProfScope pb(c, PC_QR_SMALL, 0, (double)qs.size());
      launch_qr(dqs, (int)qs.size(), 4 * 1024, st);
    }
    if (dqh) launch_qr(dqh, (int)qr_huge.size(), 0, st);
    if (par)
      for (int b = 0; b < 4; b++)
        if (dqb[b]) c->join(1 + b);
  };
  std::vector<QrJob> qjobs;
  std::vector<double*> tauA(nj, nullptr), tauB(nj, nullptr), Mp(nj, nullptr), TA(nj, nullptr), TB(nj, nullptr);
  size_t to = 0, mo = 0;
  double fl_qr = 0;
  for (int i = 0; i < nj; i++) {
    const TruncReq& r = reqs[i];
    Mp[i] = Mbuf + mo;
    mo += (size_t)p[i] * q[i];
    for (int side = 0; side < 2; side++) {
      const bool doit = side == 0 ? qa[i] : qb[i];
      if (!doit) continue;
      const int rows = side == 0 ? r.m : r.n;
      fl_qr += 2.0 * rows * r.l * r.l;
      if (tsp[side][i] >= 0) {
        const TsLevel& L = ts[tsp[side][i]].lv[0];
        for (int ch = 0; ch < L.nch; ch++) {
          int r0, cr;
          chunk(L, ch, r0, cr);
          qjobs.push_back(QrJob{L.V + r0, cr, r.l, L.ld, L.tau + (size_t)ch * r.l, chunkT(L, ch, cr, r.l)});
        }
        continue;
      }
      double* Tf = qr_has_T(rows, r.l) ? ar.alloc((size_t)((r.l + 15) / 16) * 256) : nullptr;
      qjobs.push_back(QrJob{side == 0 ? r.A : r.B, rows, r.l, rows, tau + to, Tf});
      (side == 0 ? tauA : tauB)[i] = tau + to;
      (side == 0 ? TA : TB)[i] = Tf;
      to += r.l;
    }
  }
  auto add_copy = [](std::vector<CopyJob>& v, int64_t& tiles, double* dst, int ldd, const double* src,
                     int lds, int rows, int cols, int upper) {
    CopyJob j{};
    j.dst = dst; j.src = src; j.ldd = ldd; j.lds = lds; j.rows = rows; j.cols = cols;
    j.coef = 1.0; j.upper = upper; j.tile0 = tiles;
    tiles += (int64_t)((rows + 31) / 32) * ((cols + 31) / 32);
    v.push_back(j);
  };
  c->prof_note(shapes);
  {
    ProfScope ps(c, PC_QR, fl_qr, 0);
    launch_qr_set(qjobs);
    // TSQR upper levels: stack the chunk R's, QR the stack
    for (size_t lvl = 1; lvl < maxdepth; lvl++) {
      ProfScope pt(c, PC_TSQR, 0, 0);
      std::vector<CopyJob> cj;
      std::vector<QrJob> qj;
      int64_t tiles = 0;
      for (const TsPlan& P : ts) {
        if (P.lv.size() <= lvl) continue;
        const TsLevel &D = P.lv[lvl - 1], &U = P.lv[lvl];
        for (int ch = 0; ch < D.nch; ch++) {
          int r0, cr;
          chunk(D, ch, r0, cr);
          add_copy(cj, tiles, U.V + (size_t)ch * P.l, U.ld, D.V + r0, D.ld, P.l, P.l, 1);
        }
        for (int ch = 0; ch < U.nch; ch++) {
          int r0, cr;
          chunk(U, ch, r0, cr);
          qj.push_back(QrJob{U.V + r0, cr, P.l, U.ld, U.tau + (size_t)ch * P.l, chunkT(U, ch, cr, P.l)});
        }
      }
      launch_copy_mapped(ar.upload_t(cj), (int)cj.size(), ar.tile_map_t(cj, tiles), tiles, st);
      launch_qr_set(qj);
    }
    HM_CHECK_LAUNCH();
  }
  // --- M = op(A) op(B)^T, stored in its TALL orientation Mt (L x c): Mt = M if
  // p >= q, else Mt = M^T (then the SVD's "left" side is the B side).
  std::vector<GemmJob> gj;
  gj.reserve(nj);
  int64_t tiles = 0;
  double fl_m = 0;
  std::vector<char> tallM(nj);
  for (int i = 0; i < nj; i++) {
    const TruncReq& r = reqs[i];
    tallM[i] = p[i] >= q[i];
    if (p[i] == 0 || q[i] == 0) continue;
    GemmJob g{};
    // R factor source of each side: the factor itself, or a TSQR plan's last level
    const double* ra = r.A;
    const double* rb = r.B;
    int lda_ = r.m, ldb_ = r.n;
    if (tsp[0][i] >= 0) { ra = ts[tsp[0][i]].lv.back().V; lda_ = ts[tsp[0][i]].lv.back().ld; }
    if (tsp[1][i] >= 0) { rb = ts[tsp[1][i]].lv.back().V; ldb_ = ts[tsp[1][i]].lv.back().ld; }
    if (tallM[i]) {
      g.A = ra; g.lda = lda_; g.maskA = qa[i];
      g.B = rb; g.ldb = ldb_; g.maskB = qb[i];
      g.m = p[i]; g.n = q[i]; g.ldc = p[i];
    } else {
      g.A = rb; g.lda = ldb_; g.maskA = qb[i];
      g.B = ra; g.ldb = lda_; g.maskB = qa[i];
      g.m = q[i]; g.n = p[i]; g.ldc = q[i];
    }
    g.transA = 0; g.transB = 1;
    g.C = Mp[i];
    g.k = r.l;
    g.alpha = 1.0; g.beta = 0.0;
    g.tile0 = tiles;
    tiles += (int64_t)((g.m + 63) / 64) * ((g.n + 63) / 64);
    fl_m += 2.0 * p[i] * q[i] * r.l;
    gj.push_back(g);
  }
  c->prof_note(shapes);
  {
    ProfScope ps(c, PC_GEMM_M, fl_m, 0);
    launch_gemm_mapped(ar.upload_t(gj), (int)gj.size(), ar.tile_map_t(gj, tiles), tiles, st);
    HM_CHECK_LAUNCH();
  }
  if (const char* dm = std::getenv("HM_DUMP_M")) {   // diagnostics: first job's M (tall orientation)
    const size_t cnt = (size_t)std::max(p[0], q[0]) * std::min(p[0], q[0]);
    std::vector<double> h(cnt);
    HM_CUDA(cudaStreamSynchronize(st));
    HM_CUDA(cudaMemcpy(h.data(), Mp[0], cnt * sizeof(double), cudaMemcpyDeviceToHost));
    if (FILE* f = std::fopen(dm, "wb")) {
      std::fwrite(h.data(), sizeof(double), cnt, f);
      std::fclose(f);
    }
  }
  // --- SVD jobs; matrices too large for shared memory are first reduced by an
  // unpivoted blocked QR (Mt = Q1 R1) and the SVD kernel works on R1 (c x c).
  std::vector<SvdJob> sj[5];   // 3 shared-memory buckets, global workspace, spill mode
  std::vector<SvdJob> sj13;    // the part of the 26 K bucket that fits 13 K doubles
  int caps[4] = {3 * 1024, 8 * 1024, 26 * 1024, 0};
  double fl_svd = 0, fl_b[5] = {0, 0, 0, 0, 0};
  const char* dump = std::getenv("HM_DUMP_JOBS");
  int* d_sw = dump ? static_cast<int*>(ar.alloc_bytes(sizeof(int) * (nj + 1))) : nullptr;
  std::vector<int> bucket_of(nj);
  std::vector<char> preqr(nj, 0);
  std::vector<double*> tauM(nj, nullptr), TM(nj, nullptr);
  std::vector<QrJob> pq[4];
  const int pqcap[4] = {6 * 1024, 12 * 1024, 24 * 1024, 24 * 1024};
  for (int i = 0; i < nj; i++) {
    const TruncReq& r = reqs[i];
    const int L = std::max(p[i], q[i]), cc = std::min(p[i], q[i]);
    const int64_t full = svd_smem_need(L, cc);
    static const bool use_preqr = [] { const char* e = std::getenv("HM_PREQR"); return !(e && e[0] == '0'); }();
    if (use_preqr && full > caps[2] && L > cc && L <= 24 * 1024) {
      preqr[i] = 1;
      tauM[i] = ar.alloc(cc + 1);
      const int b = L <= 384 ? 0 : (L <= 768 ? 1 : (L <= 1536 ? 2 : 3));
      if (L <= 1536) TM[i] = ar.alloc((size_t)((cc + 15) / 16) * 256);
      pq[b].push_back(QrJob{Mp[i], L, cc, L, tauM[i], TM[i]});
    }
  }
  {
    ProfScope ps(c, PC_PREQR, 0, 0);
    for (int b = 0; b < 4; b++)
      if (!pq[b].empty()) {
        prep_bucket(pq[b], b);
        launch_bucket(pq[b], ar.upload_t(pq[b]), b, pqcap[b], st);
      }
    HM_CHECK_LAUNCH();
  }
  for (int i = 0; i < nj; i++) {
    const TruncReq& r = reqs[i];
    const int L = std::max(p[i], q[i]), cc = std::min(p[i], q[i]);
    SvdJob s{};
    s.nsweep = d_sw ? d_sw + i : nullptr;
    s.M = Mp[i];
    s.ldm = std::max(L, 1);
    s.p = preqr[i] ? cc : L;
    s.q = cc;
    s.maskM = preqr[i];
    // left (orthonormal U_k) / right (V_k S_k) outputs of the tall matrix
    double* lo = tallM[i] ? r.Aout : r.Bout;
    double* ro = tallM[i] ? r.Bout : r.Aout;
    const int lrows = tallM[i] ? r.m : r.n, rrows = tallM[i] ? r.n : r.m;
    s.Aout = lo; s.lda = lrows; s.ma = lrows;
    s.Bout = ro; s.ldb = rrows; s.nb = rrows;
    s.rank = r.d_rank;
    s.sigma = r.d_sigma;
    const int Ls = s.p;
    const int64_t need = svd_smem_need(Ls, cc);
    const int cap = bucket_cap(need);
    fl_svd += 22.0 * (double)cc * cc * cc;
    int b = 3;
    for (int k = 0; k < 3; k++)
      if (cap == caps[k]) { b = k; break; }
    if (b == 3 && svd_spill_fits(Ls, cc)) b = 4;
    fl_b[b] += 22.0 * (double)cc * cc * cc;
    bucket_of[i] = b;
    if (b >= 3) s.work = ar.alloc((size_t)need);
    if (b == 2 && need <= 13 * 1024) sj13.push_back(s);   // two CTAs per SM (104 KB)
    else sj[b].push_back(s);
  }
  c->prof_note(shapes);
  {
    ProfScope ps(c, PC_SVD, fl_svd, 0);
    const SvdJob* dsj[5];
    int used = 0;
    for (int b = 0; b < 5; b++) {
      dsj[b] = sj[b].empty() ? nullptr : ar.upload_t(sj[b]);
      used += dsj[b] ? 1 : 0;
    }
    // few matrices (latency-bound steps): one launch, so that they run concurrently
    if (!sj13.empty() && sj13.size() + sj[2].size() < 296) {
      sj[2].insert(sj[2].end(), sj13.begin(), sj13.end());
      sj13.clear();
      dsj[2] = ar.upload_t(sj[2]);
    }
    const SvdJob* d13 = sj13.empty() ? nullptr : ar.upload_t(sj13);   // (uploads before any fork)
    used = d13 ? 1 : 0;
    for (int b = 0; b < 5; b++) used += dsj[b] ? 1 : 0;
    const bool par = used > 1 && c->multi_stream();
    for (int b = 4; b >= 0; b--) {   // the largest problems first; spill mode shares the global bucket's stream
      if (!dsj[b]) continue;
      const int sb_i = b == 4 ? 3 : b;
      cudaStream_t sb = par ? c->fork(1 + sb_i) : st;
      ProfScope pb(c, PC_SVD_B0 + sb_i, fl_b[b], (double)sj[b].size(), sb);
      if (b == 4) launch_svd_spill(dsj[b], (int)sj[b].size(), eps, sb);
      else launch_svd(dsj[b], (int)sj[b].size(), eps, caps[b], sb);
    }
    if (d13) {
      cudaStream_t sb = par ? c->fork(1 + 2) : st;
      ProfScope pb(c, PC_SVD_B0 + 2, 0, (double)sj13.size(), sb);
      launch_svd(d13, (int)sj13.size(), eps, 13 * 1024, sb);
    }
    if (par)
      for (int b = 0; b < 4; b++)
        if (dsj[b] || (b == 3 && dsj[4]) || (b == 2 && !sj13.empty())) c->join(1 + b);
    HM_CHECK_LAUNCH();
  }
  if (dump) {
    std::vector<int> sw(nj);
    HM_CUDA(cudaStreamSynchronize(st));
    HM_CUDA(cudaMemcpy(sw.data(), d_sw, sizeof(int) * nj, cudaMemcpyDeviceToHost));
    FILE* f = std::fopen(dump, "a");
    if (f) {
      for (int i = 0; i < nj; i++)
        std::fprintf(f, "%d %d %d %d %d %d %d\n", reqs[i].m, reqs[i].n, reqs[i].l, p[i], q[i], sw[i],
                     bucket_of[i]);
      std::fprintf(f, "# batch %d\n", nj);
      std::fclose(f);
    }
  }
  // --- apply Q1 (pre-QR of Mt) to the left output, then the stack's Q_A / Q_B
  std::vector<ApplyQJob> aq1, aq;
  for (int i = 0; i < nj; i++) {
    const TruncReq& r = reqs[i];
    if (preqr[i]) {
      const int L = std::max(p[i], q[i]), cc = std::min(p[i], q[i]);
      double* lo = tallM[i] ? r.Aout : r.Bout;
      const int lrows = tallM[i] ? r.m : r.n;
      aq1.push_back(ApplyQJob{Mp[i], tauM[i], L, cc, L, lo, lrows, cc, r.d_rank, TM[i]});
    }
    for (int side = 0; side < 2; side++) {
      if (!(side == 0 ? qa[i] : qb[i])) continue;
      if (tsp[side][i] >= 0) {   // level 0 of a TSQR plan: one job per chunk
        const TsLevel& L = ts[tsp[side][i]].lv[0];
        for (int ch = 0; ch < L.nch; ch++) {
          int r0, cr;
          chunk(L, ch, r0, cr);
          aq.push_back(ApplyQJob{L.V + r0, L.tau + (size_t)ch * r.l, cr, r.l, L.ld, L.X + r0, L.ldx,
                                 trunc_kcap(r.m, r.n, r.l), r.d_rank, chunkT(L, ch, cr, r.l)});
        }
      } else if (side == 0) {
        aq.push_back(ApplyQJob{r.A, tauA[i], r.m, r.l, r.m, r.Aout, r.m, trunc_kcap(r.m, r.n, r.l), r.d_rank, TA[i]});
      } else {
        aq.push_back(ApplyQJob{r.B, tauB[i], r.n, r.l, r.n, r.Bout, r.n, trunc_kcap(r.m, r.n, r.l), r.d_rank, TB[i]});
      }
    }
  }
  c->prof_note(shapes);
  {
    ProfScope ps(c, PC_APPLYQ, 0, 0);
    auto cmax = [](const std::vector<ApplyQJob>& v) {
      int m = 0;
      for (const ApplyQJob& j : v) m = std::max(m, j.c);
      return m;
    };
    // jobs with compact-WY T factors and <= 1536 rows: panel-wise DMMA kernel
    // (all columns of X per pass over a panel); the others: one warp per column
    static const int aq_dmma = [] { const char* e = std::getenv("HM_APPLYQ_DMMA"); return e ? std::atoi(e) : 1; }();
    auto launch_applyq_split = [&](std::vector<ApplyQJob>& v) {
      if (v.empty()) return;
      std::vector<ApplyQJob> fast, slow;
      int mm = 0;
      for (const ApplyQJob& j : v) {
        if (aq_dmma && j.T && j.m <= 1536) { fast.push_back(j); mm = std::max(mm, j.m); }
        else slow.push_back(j);
      }
      if (!fast.empty()) launch_applyq_dmma(ar.upload_t(fast), (int)fast.size(), cmax(fast), mm, st);
      if (!slow.empty()) launch_applyq(ar.upload_t(slow), (int)slow.size(), cmax(slow), st);
    };
    launch_applyq_split(aq1);
    if (!ts.empty()) {
      // TSQR: X_top[0:l] = output[0:l] (the SVD's factor), zeros below; then per
      // level (top down) X_j <- blockdiag(Q_j) X_j and scatter its l-row blocks
      // to the chunk heads of X_{j-1} (X_0 = the output itself, whose rows
      // below each chunk head are already zero).
      ProfScope pt(c, PC_TSQR, 0, 0);
      HM_CUDA(cudaMemsetAsync(xbuf, 0, xslab * sizeof(double), st));
      std::vector<CopyJob> cj;
      int64_t tiles = 0;
      for (const TsPlan& P : ts)
        add_copy(cj, tiles, P.lv.back().X, P.lv.back().ldx, P.lv[0].X, P.lv[0].ldx, P.l, P.kcap, 0);
      launch_copy_mapped(ar.upload_t(cj), (int)cj.size(), ar.tile_map_t(cj, tiles), tiles, st);
      for (size_t lvl = maxdepth - 1; lvl >= 1; lvl--) {
        std::vector<ApplyQJob> tq;
        cj.clear();
        tiles = 0;
        for (const TsPlan& P : ts) {
          if (P.lv.size() <= lvl) continue;
          const TsLevel &U = P.lv[lvl], &D = P.lv[lvl - 1];
          const int* rk = reqs[P.job].d_rank;
          for (int ch = 0; ch < U.nch; ch++) {
            int r0, cr;
            chunk(U, ch, r0, cr);
            tq.push_back(ApplyQJob{U.V + r0, U.tau + (size_t)ch * P.l, cr, P.l, U.ld, U.X + r0, U.ldx, P.kcap, rk,
                                   chunkT(U, ch, cr, P.l)});
          }
          for (int ch = 0; ch < D.nch; ch++) {
            int r0, cr;
            chunk(D, ch, r0, cr);
            add_copy(cj, tiles, D.X + r0, D.ldx, U.X + (size_t)ch * P.l, U.ldx, P.l, P.kcap, 0);
          }
        }
        launch_applyq_split(tq);
        launch_copy_mapped(ar.upload_t(cj), (int)cj.size(), ar.tile_map_t(cj, tiles), tiles, st);
      }
    }
    launch_applyq_split(aq);
    HM_CHECK_LAUNCH();
  }
}

}  // namespace hm
