// hm_build: H-matrix approximation of the BEM-like kernel matrix on the
// device (not part of the timed hot path).
//   * trees on the host (hm_tree.cpp),
//   * inadmissible leaves: exact entries (k_gen),
//   * admissible leaves: entries generated in HBM, then
//       min(m,n) <= 64 : TRUNC_eps of the exact block (stack G_b I^T),
//       otherwise      : randomized range finder (r = 64 columns, one power
//                        step), CERTIFIED by the directly computed residual
//                        ||G_b - Q W^T||_F <= 1e-12 ||G_b||_F (r doubles on
//                        failure), then TRUNC_eps(Q, W).
// Matrix-vector products with the H-matrix (hm_matvec_thin, Fig. 1) are here
// too.
#include <algorithm>
#include <cmath>
#include <numeric>

#include "hm_internal.h"

namespace hm {

namespace {

struct Blk {
  int b, m, n, r0, c0;
};

int64_t gen_tiles(int m, int n) { return (int64_t)((m + 31) / 32) * ((n + 31) / 32); }

void push_gemm(std::vector<GemmJob>& v, int64_t& tiles, const double* A, int lda, int ta,
               const double* B, int ldb, int tb, double* C, int ldc, int m, int n, int k,
               double alpha, double beta) {
  GemmJob g{};
  g.A = A; g.lda = lda; g.transA = ta;
  g.B = B; g.ldb = ldb; g.transB = tb;
  g.C = C; g.ldc = ldc;
  g.m = m; g.n = n; g.k = k;
  g.alpha = alpha; g.beta = beta;
  g.tile0 = tiles;
  tiles += (int64_t)((m + 63) / 64) * ((n + 63) / 64);
  v.push_back(g);
}

}  // namespace

Mat* build_matrix(Ctx* c, const double* pts, const double* area, const double* nrm, int64_t n, int kernel,
                  int leaf_size, double eta, double eps, int64_t* perm_out) {
  if (kernel == HM_KERNEL_DLP && !nrm) throw Error(HM_EINVAL, "hm_build: the double-layer kernel needs normals");
  std::shared_ptr<Tree> T = build_trees(pts, n, leaf_size, eta);
  if (perm_out) std::copy(T->perm.begin(), T->perm.end(), perm_out);
  cudaStream_t st = c->stream;
  Arena geo(c);
  double* dx = geo.alloc(3 * (size_t)n);
  double* dw = geo.alloc((size_t)n);
  int64_t* dperm = static_cast<int64_t*>(geo.alloc_bytes(sizeof(int64_t) * n));
  HM_CUDA(cudaMemcpyAsync(dx, pts, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, st));
  HM_CUDA(cudaMemcpyAsync(dw, area, sizeof(double) * n, cudaMemcpyHostToDevice, st));
  double* dn = nullptr;
  if (nrm) {
    dn = geo.alloc(3 * (size_t)n);
    HM_CUDA(cudaMemcpyAsync(dn, nrm, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, st));
  }
  HM_CUDA(cudaMemcpyAsync(dperm, T->perm.data(), sizeof(int64_t) * n, cudaMemcpyHostToDevice, st));

  auto* M = new Mat;
  M->tree = T;
  M->kernel = kernel;
  const int nb = T->nblocks();
  M->rank.assign(nb, 0);
  M->pA.assign(nb, nullptr);
  M->pB.assign(nb, nullptr);
  try {
    // ---------------- inadmissible leaves: exact entries
    std::vector<Blk> dense, adm;
    size_t nd = 0;
    for (int b = 0; b < nb; b++) {
      const int m = T->cl_size[T->bl_row[b]], nn = T->cl_size[T->bl_col[b]];
      const Blk k{b, m, nn, T->cl_start[T->bl_row[b]], T->cl_start[T->bl_col[b]]};
      if (T->bl_kind[b] == HM_BLOCK_DENSE) { dense.push_back(k); nd += (size_t)m * nn; }
      else if (T->bl_kind[b] == HM_BLOCK_ADM) adm.push_back(k);
    }
    double* dp = static_cast<double*>(c->dmalloc((nd + 1) * sizeof(double)));
    M->dpool = {dp, (nd + 1) * sizeof(double)};
    {
      Arena ar(c);
      std::vector<GenJob> gj;
      int64_t tiles = 0;
      size_t off = 0;
      for (auto& k : dense) {
        M->pA[k.b] = dp + off;
        gj.push_back(GenJob{dp + off, k.m, k.m, k.n, k.r0, k.c0, tiles});
        tiles += gen_tiles(k.m, k.n);
        off += (size_t)k.m * k.n;
      }
      ProfScope ps(c, PC_GEN, 0, 8.0 * nd);
      launch_gen(ar.upload(gj), (int)gj.size(), tiles, dx, dw, dn, dperm, kernel, st);
      HM_CHECK_LAUNCH();
      HM_CUDA(cudaStreamSynchronize(st));
    }
    // ---------------- admissible leaves, in memory-bounded chunks
    std::sort(adm.begin(), adm.end(), [](const Blk& a, const Blk& b) {
      return (int64_t)a.m * a.n > (int64_t)b.m * b.n;
    });
    Arena outs(c);   // per-block truncated factors (compacted at the end)
    std::vector<double*> oA(nb, nullptr), oB(nb, nullptr);
    std::vector<int> ok(nb, 0);
    const size_t budget = (size_t)4 << 30;   // generated entries per chunk (32 GB)
    size_t i0 = 0;
    int retry_r = 0;
    std::vector<Blk> pending_retry;
    while (i0 < adm.size() || !pending_retry.empty()) {
      std::vector<Blk> chunk;
      int r = 64;
      if (!pending_retry.empty()) {
        chunk.swap(pending_retry);
        retry_r = retry_r ? retry_r * 2 : 128;
        r = retry_r;
      } else {
        size_t used = 0;
        while (i0 < adm.size() && (chunk.empty() || used + (size_t)adm[i0].m * adm[i0].n <= budget)) {
          used += (size_t)adm[i0].m * adm[i0].n;
          chunk.push_back(adm[i0++]);
        }
      }
      Arena ar(c);
      size_t gtot = 0;
      for (auto& k : chunk) gtot += (size_t)k.m * k.n;
      double* G = ar.alloc(gtot + 1);
      std::vector<double*> Gp(chunk.size());
      {
        std::vector<GenJob> gj;
        int64_t tiles = 0;
        size_t off = 0;
        for (size_t i = 0; i < chunk.size(); i++) {
          Gp[i] = G + off;
          gj.push_back(GenJob{G + off, chunk[i].m, chunk[i].m, chunk[i].n, chunk[i].r0, chunk[i].c0, tiles});
          tiles += gen_tiles(chunk[i].m, chunk[i].n);
          off += (size_t)chunk[i].m * chunk[i].n;
        }
        ProfScope ps(c, PC_GEN, 0, 8.0 * gtot);
        launch_gen(ar.upload(gj), (int)gj.size(), tiles, dx, dw, dn, dperm, kernel, st);
        HM_CHECK_LAUNCH();
      }
      // small blocks: TRUNC of the exact block;  large: randomized + certificate
      std::vector<size_t> small, large;
      for (size_t i = 0; i < chunk.size(); i++) {
        if (std::min(chunk[i].m, chunk[i].n) <= std::max(64, r)) small.push_back(i);
        else large.push_back(i);
      }
      std::vector<TruncReq> reqs;
      std::vector<int> req_blk;
      int* d_rank = static_cast<int*>(ar.alloc_bytes(sizeof(int) * (chunk.size() + 1)));
      // ---- small: stack (G, I_n) if m >= n, else (I_m, G^T)
      {
        std::vector<CopyJob> cj;
        int64_t ct = 0;
        for (size_t i : small) {
          const Blk& k = chunk[i];
          const int l = std::min(k.m, k.n);
          double* A = ar.alloc((size_t)k.m * l);
          double* B = ar.alloc((size_t)k.n * l);
          HM_CUDA(cudaMemsetAsync(A, 0, sizeof(double) * k.m * l, st));
          HM_CUDA(cudaMemsetAsync(B, 0, sizeof(double) * k.n * l, st));
          CopyJob j{};
          if (k.m >= k.n) {
            j = CopyJob{A, Gp[i], k.m, k.m, k.m, k.n, 0, 0, 0, 1.0, ct};
            ct += gen_tiles(k.m, k.n);
            cj.push_back(j);
            j = CopyJob{B, nullptr, k.n, 0, k.n, k.n, 0, 1, 0, 1.0, ct};
            ct += gen_tiles(k.n, k.n);
            cj.push_back(j);
          } else {
            j = CopyJob{A, nullptr, k.m, 0, k.m, k.m, 0, 1, 0, 1.0, ct};
            ct += gen_tiles(k.m, k.m);
            cj.push_back(j);
            j = CopyJob{B, Gp[i], k.n, k.m, k.n, k.m, 1, 0, 0, 1.0, ct};
            ct += gen_tiles(k.n, k.m);
            cj.push_back(j);
          }
          const int kcap = trunc_kcap(k.m, k.n, l);
          double* Ao = outs.alloc((size_t)k.m * std::max(kcap, 1));
          double* Bo = outs.alloc((size_t)k.n * std::max(kcap, 1));
          reqs.push_back(TruncReq{k.m, k.n, l, A, B, Ao, Bo, d_rank + reqs.size(), nullptr});
          req_blk.push_back((int)i);
        }
        if (!cj.empty()) {
          launch_copy(ar.upload(cj), (int)cj.size(), ct, st);
          HM_CHECK_LAUNCH();
        }
      }
      // ---- large: randomized range finder with one power step
      std::vector<size_t> certified;
      if (!large.empty()) {
        const size_t L = large.size();
        std::vector<double*> Om(L), Y(L), Z(L), W(L), tauY(L), tauZ(L);
        for (size_t a = 0; a < L; a++) {
          const Blk& k = chunk[large[a]];
          Om[a] = ar.alloc((size_t)k.n * r);
          Y[a] = ar.alloc((size_t)k.m * r);
          Z[a] = ar.alloc((size_t)k.n * r);
          W[a] = ar.alloc((size_t)k.n * r);
          tauY[a] = ar.alloc(r);
          tauZ[a] = ar.alloc(r);
          launch_randn(Om[a], (int64_t)k.n * r, 0x1703908500000000ULL ^ ((uint64_t)k.b << 20) ^ (uint64_t)r, st);
        }
        auto gemm_all = [&](int which) {
          // 0: Y = G Om ; 1: Z = G^T Q(Y) ; 2: Y = G Q(Z) ; 3: W = G^T Q(Y)
          std::vector<GemmJob> gj;
          int64_t tiles = 0;
          for (size_t a = 0; a < L; a++) {
            const Blk& k = chunk[large[a]];
            if (which == 0) push_gemm(gj, tiles, Gp[large[a]], k.m, 0, Om[a], k.n, 0, Y[a], k.m, k.m, r, k.n, 1.0, 0.0);
            if (which == 1) push_gemm(gj, tiles, Gp[large[a]], k.m, 1, Y[a], k.m, 0, Z[a], k.n, k.n, r, k.m, 1.0, 0.0);
            if (which == 2) push_gemm(gj, tiles, Gp[large[a]], k.m, 0, Z[a], k.n, 0, Y[a], k.m, k.m, r, k.n, 1.0, 0.0);
            if (which == 3) push_gemm(gj, tiles, Gp[large[a]], k.m, 1, Y[a], k.m, 0, W[a], k.n, k.n, r, k.m, 1.0, 0.0);
          }
          ProfScope ps(c, PC_BUILD_GEMM, 0, 0);
          launch_gemm(ar.upload(gj), (int)gj.size(), tiles, st);
          HM_CHECK_LAUNCH();
        };
        // orthonormal basis in place: QR(X) then X <- Q [I; 0]
        auto orth_all = [&](std::vector<double*>& X, std::vector<double*>& tau, bool rows_m) {
          std::vector<QrJob> qj;
          std::vector<double*> V(L);
          for (size_t a = 0; a < L; a++) {
            const Blk& k = chunk[large[a]];
            const int rows = rows_m ? k.m : k.n;
            qj.push_back(QrJob{X[a], rows, r, rows, tau[a], nullptr});
          }
          launch_qr(ar.upload(qj), (int)qj.size(), 0, st);
          HM_CHECK_LAUNCH();
          std::vector<CopyJob> cj;
          int64_t ct = 0;
          std::vector<ApplyQJob> aq;
          for (size_t a = 0; a < L; a++) {
            const Blk& k = chunk[large[a]];
            const int rows = rows_m ? k.m : k.n;
            V[a] = ar.alloc((size_t)rows * r);
            HM_CUDA(cudaMemcpyAsync(V[a], X[a], sizeof(double) * rows * r, cudaMemcpyDeviceToDevice, st));
            HM_CUDA(cudaMemsetAsync(X[a], 0, sizeof(double) * rows * r, st));
            cj.push_back(CopyJob{X[a], nullptr, rows, 0, rows, r, 0, 1, 0, 1.0, ct});
            ct += gen_tiles(rows, r);
            aq.push_back(ApplyQJob{V[a], tau[a], rows, r, rows, X[a], rows, r, nullptr, nullptr});
          }
          launch_copy(ar.upload(cj), (int)cj.size(), ct, st);
          launch_applyq(ar.upload(aq), (int)aq.size(), r, st);
          HM_CHECK_LAUNCH();
        };
        gemm_all(0);
        orth_all(Y, tauY, true);
        gemm_all(1);
        orth_all(Z, tauZ, false);
        gemm_all(2);
        orth_all(Y, tauY, true);
        gemm_all(3);
        // certificate: ||G - Q W^T||_F^2 <= 1e-24 ||G||_F^2 (direct residual)
        std::vector<NormJob> nj;
        for (size_t a = 0; a < L; a++) {
          const Blk& k = chunk[large[a]];
          nj.push_back(NormJob{Gp[large[a]], k.m, k.n, k.m, nullptr});
        }
        double* dn = ar.alloc(2 * L);
        launch_norm(ar.upload(nj), (int)L, dn, st);
        {
          std::vector<GemmJob> gj;
          int64_t tiles = 0;
          for (size_t a = 0; a < L; a++) {
            const Blk& k = chunk[large[a]];
            push_gemm(gj, tiles, Y[a], k.m, 0, W[a], k.n, 1, Gp[large[a]], k.m, k.m, k.n, r, -1.0, 1.0);
          }
          launch_gemm(ar.upload(gj), (int)gj.size(), tiles, st);
        }
        launch_norm(ar.upload(nj), (int)L, dn + L, st);
        HM_CHECK_LAUNCH();
        std::vector<double> hn(2 * L);
        HM_CUDA(cudaStreamSynchronize(st));
        HM_CUDA(cudaMemcpy(hn.data(), dn, sizeof(double) * 2 * L, cudaMemcpyDeviceToHost));
        for (size_t a = 0; a < L; a++) {
          const Blk& k = chunk[large[a]];
          if (hn[L + a] <= 1e-24 * hn[a] || r >= std::min(k.m, k.n)) {
            const int kcap = r;
            double* Ao = outs.alloc((size_t)k.m * kcap);
            double* Bo = outs.alloc((size_t)k.n * kcap);
            reqs.push_back(TruncReq{k.m, k.n, r, Y[a], W[a], Ao, Bo, d_rank + reqs.size(), nullptr});
            req_blk.push_back((int)large[a]);
          } else {
            pending_retry.push_back(k);
          }
        }
      }
      trunc_batched(c, ar, reqs, eps);
      HM_CUDA(cudaStreamSynchronize(st));
      std::vector<int> hr(reqs.size());
      if (!reqs.empty())
        HM_CUDA(cudaMemcpy(hr.data(), d_rank, sizeof(int) * reqs.size(), cudaMemcpyDeviceToHost));
      for (size_t i = 0; i < reqs.size(); i++) {
        const int b = chunk[req_blk[i]].b;
        oA[b] = reqs[i].Aout;
        oB[b] = reqs[i].Bout;
        ok[b] = hr[i];
        M->rank[b] = hr[i];
      }
      ar.release();
    }
    // ---------------- compact the admissible factors
    size_t nf = 0;
    for (auto& k : adm) nf += (size_t)(k.m + k.n) * M->rank[k.b];
    double* fp = static_cast<double*>(c->dmalloc((nf + 1) * sizeof(double)));
    M->fpool = {fp, (nf + 1) * sizeof(double)};
    {
      Arena ar(c);
      std::vector<CopyJob> cj;
      int64_t ct = 0;
      size_t off = 0;
      for (auto& k : adm) {
        const int kk = M->rank[k.b];
        M->pA[k.b] = fp + off;
        off += (size_t)k.m * kk;
        M->pB[k.b] = fp + off;
        off += (size_t)k.n * kk;
        if (kk == 0) continue;
        cj.push_back(CopyJob{M->pA[k.b], oA[k.b], k.m, k.m, k.m, kk, 0, 0, 0, 1.0, ct});
        ct += gen_tiles(k.m, kk);
        cj.push_back(CopyJob{M->pB[k.b], oB[k.b], k.n, k.n, k.n, kk, 0, 0, 0, 1.0, ct});
        ct += gen_tiles(k.n, kk);
      }
      launch_copy(ar.upload(cj), (int)cj.size(), ct, st);
      HM_CHECK_LAUNCH();
      HM_CUDA(cudaStreamSynchronize(st));
    }
    outs.release();
    geo.release();
    HM_CUDA(cudaStreamSynchronize(st));
  } catch (...) {
    M->free_all(c);
    delete M;
    throw;
  }
  return M;
}

void matvec(Ctx* c, Mat* G, int op, double alpha, const double* x, int64_t ldx, double beta, double* y,
            int64_t ldy, int ncols) {
  const Tree& T = *G->tree;
  launch_scale(y, ldy, T.n, ncols, beta, c->stream);
  if (alpha == 0.0 || ncols == 0) return;
  std::vector<LeafDesc> lt = leaf_table(*G);
  int kmax = 1;
  for (auto& l : lt) kmax = std::max(kmax, l.k);
  const int chunk = std::max(1, std::min(ncols, 4096 / kmax));
  Arena ar(c);
  LeafDesc* d = ar.upload(lt);
  ProfScope ps(c, PC_MATVEC, 0, 0);
  // op -> (transpose, part): G, G^T, unit-lower L, upper R, Cholesky L, L^T
  static const int tr_of[6] = {0, 1, 0, 0, 0, 1};
  static const int part_of[6] = {0, 0, 1, 2, 3, 4};
  for (int j0 = 0; j0 < ncols; j0 += chunk) {
    const int nc = std::min(chunk, ncols - j0);
    launch_matvec_leaves(d, (int)lt.size(), tr_of[op], alpha, x + j0 * ldx, ldx, y + j0 * ldy, ldy, nc,
                         part_of[op], c->stream);
  }
  HM_CHECK_LAUNCH();
  HM_CUDA(cudaStreamSynchronize(c->stream));
}

}  // namespace hm
