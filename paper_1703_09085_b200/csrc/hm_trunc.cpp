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
  std::vector<TruncSmallJob> fb[3];
  const int fcap[3] = {4 * 1024, 10 * 1024, 26 * 1024};
  std::vector<TruncReq> rest;
  static const bool no_fused = std::getenv("HM_NO_FUSED") != nullptr;
  double fl = 0, by = 0;
  for (const TruncReq& r : reqs) {
    const int need = trunc_small_need(r.m, r.n, r.l);
    int b = -1;
    for (int k = 0; k < 3; k++)
      if (need <= fcap[k]) { b = k; break; }
    if (b < 0 || no_fused) { rest.push_back(r); continue; }
    fb[b].push_back(TruncSmallJob{r.A, r.B, r.m, r.n, r.l, r.Aout, r.Bout, r.d_rank, r.d_sigma});
    fl += trunc_flops(r.m, r.n, r.l, 0.0);   // convention flops (reform term k unknown here)
    by += trunc_bytes(r.m, r.n, r.l, 0.0);
  }
  {
    ProfScope ps(c, PC_FUSED, fl, by);
    for (int b = 0; b < 3; b++)
      if (!fb[b].empty()) launch_trunc_small(ar.upload(fb[b]), (int)fb[b].size(), eps, fcap[b], c->stream);
    HM_CHECK_LAUNCH();
  }
  trunc_general(c, ar, rest, eps);
}

static void trunc_general(Ctx* c, Arena& ar, const std::vector<TruncReq>& reqs, double eps) {
  if (reqs.empty()) return;
  cudaStream_t st = c->stream;
  const int nj = (int)reqs.size();
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
    if (r.l < r.m && r.l < r.n && (int64_t)std::min(r.m, r.n) * r.l > 12 * 1024) qa[i] = qb[i] = 1;
    p[i] = qa[i] ? r.l : r.m;
    q[i] = qb[i] ? r.l : r.n;
    if (qa[i]) tau_total += r.l;
    if (qb[i]) tau_total += r.l;
    m_total += (size_t)p[i] * q[i];
  }
  double* tau = ar.alloc(tau_total + 1);
  double* Mbuf = ar.alloc(m_total + 1);
  // --- QR jobs, bucketed by shared-memory need
  std::vector<QrJob> qr_small, qr_big, qr_glob;
  std::vector<double*> tauA(nj, nullptr), tauB(nj, nullptr), Mp(nj, nullptr);
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
      QrJob j{side == 0 ? r.A : r.B, rows, r.l, rows, tau + to, nullptr};
      (side == 0 ? tauA : tauB)[i] = tau + to;
      to += r.l;
      const int64_t need = (int64_t)rows * r.l;
      fl_qr += 2.0 * rows * r.l * r.l;
      if (need <= 4 * 1024) qr_small.push_back(j);
      else if (need <= qr_smem_capacity()) qr_big.push_back(j);
      else qr_glob.push_back(j);
    }
  }
  {
    ProfScope ps(c, PC_QR, fl_qr, 0);
    if (!qr_small.empty()) {
      ProfScope pb(c, PC_QR_SMALL, 0, (double)qr_small.size());
      launch_qr(ar.upload(qr_small), (int)qr_small.size(), 4 * 1024, st);
    }
    // blocked (compact-WY) QR, bucketed by panel height so that small panels
    // get several CTAs per SM: cap = 16 * rows doubles of shared memory
    std::vector<QrJob> qb[4], qr_huge;
    const int qcap[4] = {6 * 1024, 12 * 1024, 24 * 1024, 24 * 1024};
    for (auto* v : {&qr_big, &qr_glob})
      for (auto& j : *v) {
        if (j.m > 24 * 1024) { qr_huge.push_back(j); continue; }
        const int b = j.m <= 384 ? 0 : (j.m <= 768 ? 1 : (j.m <= 1536 ? 2 : 3));
        qb[b].push_back(j);
      }
    for (int b = 0; b < 4; b++)
      if (!qb[b].empty()) {
        ProfScope pb(c, PC_QR_B0 + b, 0, (double)qb[b].size());
        launch_qr_blocked(ar.upload(qb[b]), (int)qb[b].size(), qcap[b], st);
      }
    if (!qr_huge.empty()) launch_qr(ar.upload(qr_huge), (int)qr_huge.size(), 0, st);
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
    if (tallM[i]) {
      g.A = r.A; g.lda = r.m; g.maskA = qa[i];
      g.B = r.B; g.ldb = r.n; g.maskB = qb[i];
      g.m = p[i]; g.n = q[i]; g.ldc = p[i];
    } else {
      g.A = r.B; g.lda = r.n; g.maskA = qb[i];
      g.B = r.A; g.ldb = r.m; g.maskB = qa[i];
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
  {
    ProfScope ps(c, PC_GEMM_M, fl_m, 0);
    launch_gemm(ar.upload(gj), (int)gj.size(), tiles, st);
    HM_CHECK_LAUNCH();
  }
  // --- SVD jobs; matrices too large for shared memory are first reduced by an
  // unpivoted blocked QR (Mt = Q1 R1) and the SVD kernel works on R1 (c x c).
  std::vector<SvdJob> sj[4];
  int caps[4] = {3 * 1024, 8 * 1024, 26 * 1024, 0};
  double fl_svd = 0, fl_b[4] = {0, 0, 0, 0};
  const char* dump = std::getenv("HM_DUMP_JOBS");
  int* d_sw = dump ? static_cast<int*>(ar.alloc_bytes(sizeof(int) * (nj + 1))) : nullptr;
  std::vector<int> bucket_of(nj);
  std::vector<char> preqr(nj, 0);
  std::vector<double*> tauM(nj, nullptr);
  std::vector<QrJob> pq[4];
  const int pqcap[4] = {6 * 1024, 12 * 1024, 24 * 1024, 24 * 1024};
  for (int i = 0; i < nj; i++) {
    const TruncReq& r = reqs[i];
    const int L = std::max(p[i], q[i]), cc = std::min(p[i], q[i]);
    const int64_t full = (int64_t)L * cc + 2 * (int64_t)cc * cc + 6 * (int64_t)cc;
    if (full > caps[2] && L > cc && L <= 24 * 1024) {
      preqr[i] = 1;
      tauM[i] = ar.alloc(cc + 1);
      const int b = L <= 384 ? 0 : (L <= 768 ? 1 : (L <= 1536 ? 2 : 3));
      pq[b].push_back(QrJob{Mp[i], L, cc, L, tauM[i], nullptr});
    }
  }
  {
    ProfScope ps(c, PC_PREQR, 0, 0);
    for (int b = 0; b < 4; b++)
      if (!pq[b].empty()) launch_qr_blocked(ar.upload(pq[b]), (int)pq[b].size(), pqcap[b], st);
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
    s.flip = tallM[i] ? 0 : 1;   // keep Fig. 2's convention: the A-side factor is orthonormal
    // left (orthonormal U_k) / right (V_k S_k) outputs of the tall matrix
    double* lo = tallM[i] ? r.Aout : r.Bout;
    double* ro = tallM[i] ? r.Bout : r.Aout;
    const int lrows = tallM[i] ? r.m : r.n, rrows = tallM[i] ? r.n : r.m;
    s.Aout = lo; s.lda = lrows; s.ma = lrows;
    s.Bout = ro; s.ldb = rrows; s.nb = rrows;
    s.rank = r.d_rank;
    s.sigma = r.d_sigma;
    const int Ls = s.p;
    const int64_t need = (int64_t)Ls * cc + 2 * (int64_t)cc * cc + 6 * (int64_t)cc;
    const int cap = bucket_cap(need);
    fl_svd += 22.0 * (double)cc * cc * cc;
    int b = 3;
    for (int k = 0; k < 3; k++)
      if (cap == caps[k]) { b = k; break; }
    fl_b[b] += 22.0 * (double)cc * cc * cc;
    bucket_of[i] = b;
    if (b == 3) s.work = ar.alloc((size_t)need);
    sj[b].push_back(s);
  }
  {
    ProfScope ps(c, PC_SVD, fl_svd, 0);
    for (int b = 0; b < 4; b++) {
      if (sj[b].empty()) continue;
      ProfScope pb(c, PC_SVD_B0 + b, fl_b[b], (double)sj[b].size());
      launch_svd(ar.upload(sj[b]), (int)sj[b].size(), eps, caps[b], st);
    }
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
      aq1.push_back(ApplyQJob{Mp[i], tauM[i], L, cc, L, lo, lrows, 0, r.d_rank});
    }
    if (qa[i]) aq.push_back(ApplyQJob{r.A, tauA[i], r.m, r.l, r.m, r.Aout, r.m, 0, r.d_rank});
    if (qb[i]) aq.push_back(ApplyQJob{r.B, tauB[i], r.n, r.l, r.n, r.Bout, r.n, 0, r.d_rank});
  }
  {
    ProfScope ps(c, PC_APPLYQ, 0, 0);
    if (!aq1.empty()) launch_applyq(ar.upload(aq1), (int)aq1.size(), st);
    if (!aq.empty()) launch_applyq(ar.upload(aq), (int)aq.size(), st);
    HM_CHECK_LAUNCH();
  }
}

}  // namespace hm
