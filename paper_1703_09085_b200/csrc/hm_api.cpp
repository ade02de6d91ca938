// C-ABI entry points of libhm (include/hm.h).  Every entry point catches
// all exceptions and converts them to hm_status + hm_last_error().
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <new>

#include "hm_internal.h"

using namespace hm;

struct hm_ctx_s {
  Ctx c;
};
struct hm_mat_s {
  Mat m;
};

namespace {
template <class F>
hm_status guard(hm_ctx ctx, F&& f) {
  try {
    f();
    return HM_OK;
  } catch (const Error& e) {
    if (ctx) ctx->c.err = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    if (ctx) ctx->c.err = "host allocation failed";
    return HM_ENOMEM;
  } catch (const std::exception& e) {
    if (ctx) ctx->c.err = e.what();
    return HM_EINVAL;
  }
}

void set_device(Ctx& c) { HM_CUDA(cudaSetDevice(c.device)); }

std::shared_ptr<Tree> tree_from_desc(const hm_host_desc* d) {
  auto T = std::make_shared<Tree>();
  T->n = d->n;
  const int nc = d->nclusters, nb = d->nblocks;
  if (nc <= 0 || nb <= 0) throw Error(HM_EINVAL, "hm_import: empty trees");
  T->cl_start.assign(d->cl_start, d->cl_start + nc);
  T->cl_size.assign(d->cl_size, d->cl_size + nc);
  T->cl_son0.assign(d->cl_son0, d->cl_son0 + nc);
  T->cl_nsons.assign(d->cl_nsons, d->cl_nsons + nc);
  T->cl_level.assign(d->cl_level, d->cl_level + nc);
  if (d->cl_bbox) T->cl_bbox.assign(d->cl_bbox, d->cl_bbox + 6 * (size_t)nc);
  T->bl_row.assign(d->bl_row, d->bl_row + nb);
  T->bl_col.assign(d->bl_col, d->bl_col + nb);
  T->bl_kind.assign(d->bl_kind, d->bl_kind + nb);
  T->bl_son0.assign(d->bl_son0, d->bl_son0 + nb);
  T->bl_nsons.assign(d->bl_nsons, d->bl_nsons + nb);
  if (d->perm) T->perm.assign(d->perm, d->perm + d->n);
  // structural validation
  for (int b = 0; b < nb; b++) {
    const int t = T->bl_row[b], s = T->bl_col[b];
    if (t < 0 || t >= nc || s < 0 || s >= nc) throw Error(HM_EINVAL, "hm_import: bad cluster id");
    const int k = T->bl_kind[b];
    if (k < 0 || k > 2) throw Error(HM_EINVAL, "hm_import: bad block kind");
    if (k == HM_BLOCK_SUB) {
      if (T->bl_nsons[b] != T->cl_nsons[t] * T->cl_nsons[s] || T->bl_son0[b] <= b ||
          T->bl_son0[b] + T->bl_nsons[b] > nb)
        throw Error(HM_EINVAL, "hm_import: inconsistent block sons");
      for (int i = 0; i < T->cl_nsons[t]; i++)
        for (int j = 0; j < T->cl_nsons[s]; j++) {
          const int sb = T->bl_son0[b] + i * T->cl_nsons[s] + j;
          if (T->bl_row[sb] != T->cl_son0[t] + i || T->bl_col[sb] != T->cl_son0[s] + j)
            throw Error(HM_EINVAL, "hm_import: block sons are not sons(t) x sons(s)");
        }
    }
  }
  T->finalize();
  return T;
}

void upload_payload(Ctx& c, Mat& M, const hm_host_desc* d) {
  const Tree& T = *M.tree;
  const int nb = T.nblocks();
  M.rank.assign(nb, 0);
  M.pA.assign(nb, nullptr);
  M.pB.assign(nb, nullptr);
  size_t nf = 0, nd = 0;
  for (int b = 0; b < nb; b++) {
    const int64_t m = T.cl_size[T.bl_row[b]], n = T.cl_size[T.bl_col[b]];
    if (T.bl_kind[b] == HM_BLOCK_ADM) {
      const int k = d->bl_rank[b];
      if (k < 0 || d->bl_off[b] < 0 || d->bl_off[b] + (m + n) * k > d->nfactors)
        throw Error(HM_EINVAL, "hm_import: factor payload out of range");
      M.rank[b] = k;
      nf += (size_t)(m + n) * k;
    } else if (T.bl_kind[b] == HM_BLOCK_DENSE) {
      if (d->bl_off[b] < 0 || d->bl_off[b] + m * n > d->ndense)
        throw Error(HM_EINVAL, "hm_import: dense payload out of range");
      nd += (size_t)m * n;
    }
  }
  double* fp = static_cast<double*>(c.dmalloc((nf + 1) * sizeof(double)));
  M.fpool = {fp, (nf + 1) * sizeof(double)};
  double* dp = static_cast<double*>(c.dmalloc((nd + 1) * sizeof(double)));
  M.dpool = {dp, (nd + 1) * sizeof(double)};
  // payload in block order and contiguous (what hm_export writes): one bulk
  // copy per pool; otherwise repack on the host first
  bool fcont = true, dcont = true;
  {
    int64_t of = 0, od = 0;
    for (int b = 0; b < nb; b++) {
      const int64_t m = T.cl_size[T.bl_row[b]], n = T.cl_size[T.bl_col[b]];
      if (T.bl_kind[b] == HM_BLOCK_ADM) {
        if (M.rank[b] > 0 && d->bl_off[b] != of) fcont = false;
        of += (m + n) * M.rank[b];
      } else if (T.bl_kind[b] == HM_BLOCK_DENSE) {
        if (d->bl_off[b] != od) dcont = false;
        od += m * n;
      }
    }
  }
  std::vector<double> hf, hd;
  if (!fcont) hf.resize(nf);
  if (!dcont) hd.resize(nd);
  size_t of = 0, od = 0;
  for (int b = 0; b < nb; b++) {
    const int64_t m = T.cl_size[T.bl_row[b]], n = T.cl_size[T.bl_col[b]];
    if (T.bl_kind[b] == HM_BLOCK_ADM) {
      const int k = M.rank[b];
      if (!fcont) std::memcpy(hf.data() + of, d->factors + d->bl_off[b], sizeof(double) * (m + n) * k);
      M.pA[b] = fp + of;
      M.pB[b] = fp + of + m * k;
      of += (m + n) * k;
    } else if (T.bl_kind[b] == HM_BLOCK_DENSE) {
      if (!dcont) std::memcpy(hd.data() + od, d->dense + d->bl_off[b], sizeof(double) * m * n);
      M.pA[b] = dp + od;
      od += m * n;
    }
  }
  if (nf)
    HM_CUDA(cudaMemcpyAsync(fp, fcont ? d->factors : hf.data(), nf * sizeof(double), cudaMemcpyHostToDevice, c.stream));
  if (nd)
    HM_CUDA(cudaMemcpyAsync(dp, dcont ? d->dense : hd.data(), nd * sizeof(double), cudaMemcpyHostToDevice, c.stream));
  HM_CUDA(cudaStreamSynchronize(c.stream));
}
}  // namespace

extern "C" {

const char* hm_version(void) { return "libhm 0.1 (sm_100a, FP64)"; }

hm_status hm_ctx_create(int device, void* cuda_stream, const hm_allocator* alloc, hm_ctx* out) {
  if (!out) return HM_EINVAL;
  hm_ctx c = new (std::nothrow) hm_ctx_s;
  if (!c) return HM_ENOMEM;
  c->c.device = device;
  c->c.stream = static_cast<cudaStream_t>(cuda_stream);
  if (alloc && alloc->alloc && alloc->free) {
    c->c.alloc = *alloc;
    c->c.has_alloc = true;
  }
  hm_status s = guard(c, [&] {
    int ndev = 0;
    HM_CUDA(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) throw Error(HM_EINVAL, "hm_ctx_create: bad device");
    set_device(c->c);
    int major = 0;
    HM_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
    if (major != 10) throw Error(HM_EUNSUPPORTED, "libhm is built for sm_100a (B200) only");
    // a PRIVATE stream-ordered pool that keeps freed allocations cached: every
    // level of hm_addmul allocates and frees its stacks, and re-mapping tens of
    // GB per level would dominate the run time.  The device's default pool (the
    // one torch and other cudaMallocAsync users see) is left untouched; the
    // private pool's memory is returned by hm_ctx_destroy.
    // HM_POOL=default: the device's default pool (profiling tools that do not
    // follow private pools); the release threshold is raised as before
    const char* pe = std::getenv("HM_POOL");
    if (!c->c.has_alloc && pe && std::string(pe) == "default") {
      cudaMemPool_t dp;
      HM_CUDA(cudaDeviceGetDefaultMemPool(&dp, device));
      uint64_t thr = UINT64_MAX;
      HM_CUDA(cudaMemPoolSetAttribute(dp, cudaMemPoolAttrReleaseThreshold, &thr));
    } else if (!c->c.has_alloc) {
      cudaMemPoolProps props{};
      props.allocType = cudaMemAllocationTypePinned;
      props.location.type = cudaMemLocationTypeDevice;
      props.location.id = device;
      HM_CUDA(cudaMemPoolCreate(&c->c.pool, &props));
      uint64_t thr = UINT64_MAX;
      HM_CUDA(cudaMemPoolSetAttribute(c->c.pool, cudaMemPoolAttrReleaseThreshold, &thr));
    }
  });
  if (s != HM_OK) {
    delete c;
    return s;
  }
  *out = c;
  return HM_OK;
}

hm_status hm_ctx_destroy(hm_ctx ctx) {
  if (!ctx) return HM_EINVAL;
  cudaSetDevice(ctx->c.device);
  cudaStreamSynchronize(ctx->c.stream);
  ctx->c.prof_collect();
  for (auto e : ctx->c.free_events) cudaEventDestroy(e);
  // every hm_mat of the context is released here (include/hm.h): handles
  // become invalid
  for (void* p : ctx->c.live) {
    auto* m = static_cast<hm_mat_s*>(p);
    m->m.free_all(&ctx->c);
    delete m;
  }
  ctx->c.live.clear();
  delete ctx;
  return HM_OK;
}

const char* hm_last_error(hm_ctx ctx) { return ctx ? ctx->c.err.c_str() : "null context"; }

hm_status hm_sync(hm_ctx ctx) {
  if (!ctx) return HM_EINVAL;
  return guard(ctx, [&] { HM_CUDA(cudaStreamSynchronize(ctx->c.stream)); });
}

hm_status hm_trim(hm_ctx ctx) {
  if (!ctx) return HM_EINVAL;
  return guard(ctx, [&] {
    set_device(ctx->c);
    ctx->c.trim();
  });
}

hm_status hm_import(hm_ctx ctx, const hm_host_desc* d, hm_mat* out) {
  if (!ctx || !d || !out) return HM_EINVAL;
  return guard(ctx, [&] {
    set_device(ctx->c);
    auto* M = new hm_mat_s;
    try {
      M->m.tree = tree_from_desc(d);
      upload_payload(ctx->c, M->m, d);
    } catch (...) {
      M->m.free_all(&ctx->c);
      delete M;
      throw;
    }
    ctx->c.live.insert(M);
    *out = M;
  });
}

static void export_impl(hm_ctx ctx, hm_mat mat, hm_host_desc* d, double* fout, double* dout, bool user) {
  {
    set_device(ctx->c);
    Mat& M = mat->m;
    const Tree& T = *M.tree;
    const int nb = T.nblocks();
    M.ex_rank.assign(nb, 0);
    M.ex_off.assign(nb, -1);
    size_t nf = 0, nd = 0;
    for (int b = 0; b < nb; b++) {
      const int64_t m = T.cl_size[T.bl_row[b]], n = T.cl_size[T.bl_col[b]];
      if (T.bl_kind[b] == HM_BLOCK_ADM) {
        M.ex_rank[b] = M.rank[b];
        M.ex_off[b] = (int64_t)nf;
        nf += (size_t)(m + n) * M.rank[b];
      } else if (T.bl_kind[b] == HM_BLOCK_DENSE) {
        M.ex_off[b] = (int64_t)nd;
        nd += (size_t)m * n;
      }
    }
    if (user) {
      if ((nf && !fout) || (nd && !dout)) throw Error(HM_EINVAL, "hm_export_into: null payload buffer");
    } else {
      M.ex_factors.reset(new double[nf + 1]);
      M.ex_dense.reset(new double[nd + 1]);
      fout = M.ex_factors.get();
      dout = M.ex_dense.get();
    }
    // gather the blocks into export order on the device (one batched copy per
    // pool), then one bulk D2H per pool
    {
      Arena ar(&ctx->c);
      double* gf = nf ? ar.alloc(nf) : nullptr;
      double* gd = nd ? ar.alloc(nd) : nullptr;
      std::vector<CopyJob> cj;
      int64_t tiles = 0;
      auto add = [&](double* dst, const double* src, int64_t cnt) {
        // a contiguous run of cnt doubles as a (1024 x ceil) column block
        const int rows = 1024;
        const int cols = (int)((cnt + rows - 1) / rows);
        const int full = (int)(cnt / rows);
        if (full > 0) {
          CopyJob j{};
          j.dst = dst; j.src = src; j.ldd = rows; j.lds = rows; j.rows = rows; j.cols = full;
          j.coef = 1.0; j.tile0 = tiles;
          tiles += (int64_t)(rows / 32) * ((full + 31) / 32);
          cj.push_back(j);
        }
        if (cols > full) {
          CopyJob j{};
          const int64_t off = (int64_t)full * rows;
          j.dst = dst + off; j.src = src + off; j.ldd = rows; j.lds = rows; j.rows = (int)(cnt - off); j.cols = 1;
          j.coef = 1.0; j.tile0 = tiles;
          tiles += (int64_t)((j.rows + 31) / 32);
          cj.push_back(j);
        }
      };
      for (int b = 0; b < nb; b++) {
        const int64_t m = T.cl_size[T.bl_row[b]], n = T.cl_size[T.bl_col[b]];
        if (T.bl_kind[b] == HM_BLOCK_ADM && M.rank[b] > 0) {
          const int64_t k = M.rank[b];
          add(gf + M.ex_off[b], M.pA[b], m * k);
          add(gf + M.ex_off[b] + m * k, M.pB[b], n * k);
        } else if (T.bl_kind[b] == HM_BLOCK_DENSE) {
          add(gd + M.ex_off[b], M.pA[b], m * n);
        }
      }
      if (!cj.empty()) launch_copy(ar.upload(cj), (int)cj.size(), tiles, ctx->c.stream);
      HM_CHECK_LAUNCH();
      if (nf) HM_CUDA(cudaMemcpyAsync(fout, gf, nf * sizeof(double), cudaMemcpyDeviceToHost, ctx->c.stream));
      if (nd) HM_CUDA(cudaMemcpyAsync(dout, gd, nd * sizeof(double), cudaMemcpyDeviceToHost, ctx->c.stream));
      HM_CUDA(cudaStreamSynchronize(ctx->c.stream));
      ar.release();
    }
    std::memset(d, 0, sizeof(*d));
    d->n = T.n;
    d->nclusters = T.nclusters();
    d->cl_start = T.cl_start.data();
    d->cl_size = T.cl_size.data();
    d->cl_son0 = T.cl_son0.data();
    d->cl_nsons = T.cl_nsons.data();
    d->cl_level = T.cl_level.data();
    d->cl_bbox = T.cl_bbox.empty() ? nullptr : T.cl_bbox.data();
    d->nblocks = nb;
    d->bl_row = T.bl_row.data();
    d->bl_col = T.bl_col.data();
    d->bl_kind = T.bl_kind.data();
    d->bl_son0 = T.bl_son0.data();
    d->bl_nsons = T.bl_nsons.data();
    d->bl_rank = M.ex_rank.data();
    d->bl_off = M.ex_off.data();
    d->factors = fout;
    d->nfactors = (int64_t)nf;
    d->dense = dout;
    d->ndense = (int64_t)nd;
    d->perm = T.perm.empty() ? nullptr : T.perm.data();
  }
}

hm_status hm_export(hm_ctx ctx, hm_mat mat, hm_host_desc* d) {
  if (!ctx || !mat || !d) return HM_EINVAL;
  return guard(ctx, [&] { export_impl(ctx, mat, d, nullptr, nullptr, false); });
}

hm_status hm_export_into(hm_ctx ctx, hm_mat mat, hm_host_desc* d, double* factors_out, double* dense_out) {
  if (!ctx || !mat || !d) return HM_EINVAL;
  return guard(ctx, [&] { export_impl(ctx, mat, d, factors_out, dense_out, true); });
}

hm_status hm_export_sizes(hm_ctx ctx, hm_mat mat, int64_t* nfactors, int64_t* ndense) {
  if (!ctx || !mat || !nfactors || !ndense) return HM_EINVAL;
  return guard(ctx, [&] {
    const Mat& M = mat->m;
    const Tree& T = *M.tree;
    int64_t nf = 0, nd = 0;
    for (int b = 0; b < T.nblocks(); b++) {
      const int64_t m = T.cl_size[T.bl_row[b]], n = T.cl_size[T.bl_col[b]];
      if (T.bl_kind[b] == HM_BLOCK_ADM) nf += (m + n) * M.rank[b];
      else if (T.bl_kind[b] == HM_BLOCK_DENSE) nd += m * n;
    }
    *nfactors = nf;
    *ndense = nd;
  });
}

hm_status hm_clone(hm_ctx ctx, hm_mat src, hm_mat* out) {
  if (!ctx || !src || !out) return HM_EINVAL;
  return guard(ctx, [&] {
    set_device(ctx->c);
    const Mat& S = src->m;
    auto* M = new hm_mat_s;
    M->m.tree = S.tree;
    M->m.rank = S.rank;
    M->m.kernel = S.kernel;
    const int nb = S.tree->nblocks();
    M->m.pA.assign(nb, nullptr);
    M->m.pB.assign(nb, nullptr);
    double* fp = static_cast<double*>(ctx->c.dmalloc(S.fpool.second));
    double* dp = static_cast<double*>(ctx->c.dmalloc(S.dpool.second));
    M->m.fpool = {fp, S.fpool.second};
    M->m.dpool = {dp, S.dpool.second};
    HM_CUDA(cudaMemcpyAsync(fp, S.fpool.first, S.fpool.second, cudaMemcpyDeviceToDevice, ctx->c.stream));
    HM_CUDA(cudaMemcpyAsync(dp, S.dpool.first, S.dpool.second, cudaMemcpyDeviceToDevice, ctx->c.stream));
    const double* f0 = static_cast<const double*>(S.fpool.first);
    const double* d0 = static_cast<const double*>(S.dpool.first);
    for (int b = 0; b < nb; b++) {
      if (S.tree->bl_kind[b] == HM_BLOCK_ADM) {
        M->m.pA[b] = fp + (S.pA[b] - f0);
        M->m.pB[b] = fp + (S.pB[b] - f0);
      } else if (S.tree->bl_kind[b] == HM_BLOCK_DENSE) {
        M->m.pA[b] = dp + (S.pA[b] - d0);
      }
    }
    ctx->c.live.insert(M);
    *out = M;
  });
}

hm_status hm_free(hm_ctx ctx, hm_mat m) {
  if (!ctx || !m) return HM_EINVAL;
  return guard(ctx, [&] {
    if (!ctx->c.live.erase(m)) throw Error(HM_EINVAL, "hm_free: matrix does not belong to this context");
    m->m.free_all(&ctx->c);
    delete m;
  });
}

hm_status hm_addmul(hm_ctx ctx, double alpha, hm_mat X, hm_mat Y, hm_mat Z, double eps) {
  if (!ctx || !X || !Y || !Z) return HM_EINVAL;
  return guard(ctx, [&] {
    set_device(ctx->c);
    addmul(&ctx->c, alpha, &X->m, &Y->m, &Z->m, eps);
  });
}

hm_status hm_build(hm_ctx ctx, const double* pts_host, const double* area_host, int64_t n, int kernel,
                   int leaf_size, double eta, double eps, hm_mat* out, int64_t* perm_host) {
  return hm_build_nrm(ctx, pts_host, area_host, nullptr, n, kernel, leaf_size, eta, eps, out, perm_host);
}

hm_status hm_build_nrm(hm_ctx ctx, const double* pts_host, const double* area_host, const double* nrm_host,
                       int64_t n, int kernel, int leaf_size, double eta, double eps, hm_mat* out,
                       int64_t* perm_host) {
  if (!ctx || !pts_host || !area_host || !out) return HM_EINVAL;
  return guard(ctx, [&] {
    set_device(ctx->c);
    if (kernel != HM_KERNEL_SLP && kernel != HM_KERNEL_SLP_SYM && kernel != HM_KERNEL_DLP)
      throw Error(HM_EINVAL, "hm_build: unknown kernel");
    if (!(eps >= 0.0)) throw Error(HM_EINVAL, "hm_build: eps must be >= 0");
    // the build's temporaries are the largest allocations of a session: if it
    // runs out of memory, the workspaces earlier operations left behind are
    // given back (hm_trim) and it is tried once more
    Mat* M = nullptr;
    try {
      M = build_matrix(&ctx->c, pts_host, area_host, nrm_host, n, kernel, leaf_size, eta, eps, perm_host);
    } catch (const Error& e) {
      if (e.code != HM_ENOMEM) throw;
      cudaGetLastError();
      ctx->c.trim(false);
      M = build_matrix(&ctx->c, pts_host, area_host, nrm_host, n, kernel, leaf_size, eta, eps, perm_host);
    }
    auto* H = new hm_mat_s;
    H->m = std::move(*M);
    delete M;
    ctx->c.live.insert(H);
    *out = H;
  });
}

hm_status hm_addmul_std(hm_ctx ctx, double alpha, hm_mat X, hm_mat Y, hm_mat Z, double eps) {
  if (!ctx || !X || !Y || !Z) return HM_EINVAL;
  return guard(ctx, [&] {
    set_device(ctx->c);
    addmul_std(&ctx->c, alpha, &X->m, &Y->m, &Z->m, eps);
  });
}

hm_status hm_solve_thin(hm_ctx ctx, hm_mat F, int op, double* x_dev, int64_t ldx, int ncols) {
  if (!ctx || !F) return HM_EINVAL;
  return guard(ctx, [&] {
    set_device(ctx->c);
    solve_thin(&ctx->c, &F->m, op, x_dev, ldx, ncols);
  });
}

hm_status hm_precond_error(hm_ctx ctx, hm_mat G, hm_mat F, int kind, int iters, uint64_t seed, double* out) {
  if (!ctx || !G || !F || !out || kind < 0 || kind > 2) return HM_EINVAL;
  return guard(ctx, [&] {
    set_device(ctx->c);
    *out = precond_error(&ctx->c, &G->m, &F->m, kind, iters, seed);
  });
}

hm_status hm_inv(hm_ctx ctx, hm_mat G, double eps) {
  if (!ctx || !G) return HM_EINVAL;
  return guard(ctx, [&] {
    set_device(ctx->c);
    double mp = 0;
    ctx->c.last = hm_stats_t{};
    invert_matrix(&ctx->c, &G->m, eps, &mp);
    ctx->c.last.min_pivot = mp;
  });
}

hm_status hm_lr(hm_ctx ctx, hm_mat G, double eps) {
  if (!ctx || !G) return HM_EINVAL;
  return guard(ctx, [&] {
    set_device(ctx->c);
    double mp = 0;
    ctx->c.last = hm_stats_t{};
    factorize(&ctx->c, &G->m, eps, false, 0.0, &mp);
    ctx->c.last.min_pivot = mp;
  });
}

hm_status hm_chol(hm_ctx ctx, hm_mat G, double eps, double shift) {
  if (!ctx || !G) return HM_EINVAL;
  return guard(ctx, [&] {
    set_device(ctx->c);
    double mp = 0;
    ctx->c.last = hm_stats_t{};
    factorize(&ctx->c, &G->m, eps, true, shift, &mp);
    ctx->c.last.min_pivot = mp;
  });
}

hm_status hm_matvec_thin(hm_ctx ctx, hm_mat G, int op, double alpha, const double* x_dev, int64_t ldx,
                         double beta, double* y_dev, int64_t ldy, int ncols) {
  if (!ctx || !G || !x_dev || !y_dev) return HM_EINVAL;
  return guard(ctx, [&] {
    set_device(ctx->c);
    if (op < HM_OP_G || op > HM_OP_LCT) throw Error(HM_EINVAL, "hm_matvec_thin: bad op");
    if (ncols < 0 || ldx < G->m.tree->n || ldy < G->m.tree->n)
      throw Error(HM_EINVAL, "hm_matvec_thin: bad leading dimension");
    matvec(&ctx->c, &G->m, op, alpha, x_dev, ldx, beta, y_dev, ldy, ncols);
  });
}

hm_status hm_stats(hm_ctx ctx, hm_mat m, hm_stats_t* out) {
  if (!ctx || !out) return HM_EINVAL;
  return guard(ctx, [&] {
    *out = ctx->c.last;
    out->kernel_launches = launch_count();
    if (!m) return;
    const Mat& M = m->m;
    const Tree& T = *M.tree;
    out->n = T.n;
    out->nclusters = T.nclusters();
    out->nblocks = T.nblocks();
    out->nadm = out->ndense = 0;
    out->depth = T.depth;
    out->max_rank = 0;
    double rs = 0;
    out->factor_doubles = out->dense_doubles = 0;
    for (int b = 0; b < T.nblocks(); b++) {
      const int64_t mm = T.cl_size[T.bl_row[b]], nn = T.cl_size[T.bl_col[b]];
      if (T.bl_kind[b] == HM_BLOCK_ADM) {
        out->nadm++;
        out->max_rank = std::max(out->max_rank, M.rank[b]);
        rs += M.rank[b];
        out->factor_doubles += (mm + nn) * M.rank[b];
      } else if (T.bl_kind[b] == HM_BLOCK_DENSE) {
        out->ndense++;
        out->dense_doubles += mm * nn;
      }
    }
    out->mean_rank = out->nadm ? rs / out->nadm : 0.0;
  });
}

hm_status hm_profile_enable(hm_ctx ctx, int on) {
  if (!ctx) return HM_EINVAL;
  ctx->c.prof = on != 0;
  if (ctx->c.prof && !ctx->c.plog)
    if (const char* f = std::getenv("HM_PROF_LOG")) ctx->c.plog = std::fopen(f, "w");
  return HM_OK;
}

hm_status hm_profile_reset(hm_ctx ctx) {
  if (!ctx) return HM_EINVAL;
  return guard(ctx, [&] {
    ctx->c.prof_collect();
    for (int i = 0; i < PC_COUNT; i++) {
      ctx->c.ms[i] = 0;
      ctx->c.launches[i] = 0;
      ctx->c.flops[i] = 0;
      ctx->c.bytes[i] = 0;
    }
  });
}

hm_status hm_profile_get(hm_ctx ctx, hm_prof_t* out) {
  if (!ctx || !out) return HM_EINVAL;
  return guard(ctx, [&] {
    ctx->c.prof_collect();
    static const char* names[PC_COUNT] = {"qr", "gemm_M", "jacobi_svd", "apply_q", "copy", "eval",
                                          "dense_add", "memset", "gen", "build_gemm", "norm", "matvec",
                                          "svd_smem3k", "svd_smem8k", "svd_smem26k", "svd_global", "qr_smem4k", "qr_blk384",
                                          "qr_blk768", "qr_blk1536", "qr_blk_big", "pre_qr_M", "trsm", "leaf_lu_chol", "trunc_fused",
                                          "tsqr_stack"};
    std::memset(out, 0, sizeof(*out));
    out->count = PC_COUNT;
    for (int i = 0; i < PC_COUNT; i++) {
      std::strncpy(out->name[i], names[i], 23);
      out->ms[i] = ctx->c.ms[i];
      out->launches[i] = ctx->c.launches[i];
      out->flops[i] = ctx->c.flops[i];
      out->bytes[i] = ctx->c.bytes[i];
    }
  });
}

hm_status hm_test_trunc_batched(hm_ctx ctx, int njobs, const int32_t* m, const int32_t* n, const int32_t* l,
                                double* a_dev, const int64_t* a_off, double* b_dev, const int64_t* b_off,
                                double* ua_dev, const int64_t* o_off, double* ub_dev, const int64_t* p_off,
                                double eps, int32_t* ranks_host, double* sigma_host) {
  if (!ctx || njobs < 0 || !ranks_host) return HM_EINVAL;
  return guard(ctx, [&] {
    set_device(ctx->c);
    Arena ar(&ctx->c);
    std::vector<TruncReq> reqs(njobs);
    int* d_rank = static_cast<int*>(ar.alloc_bytes(sizeof(int) * (njobs + 1)));
    size_t sig_total = 0;
    std::vector<size_t> sig_off(njobs);
    for (int i = 0; i < njobs; i++) {
      sig_off[i] = sig_total;
      sig_total += std::min(std::min(m[i], n[i]), l[i]) > 0 ? std::max(std::min(m[i], l[i]), 1) : 1;
    }
    double* d_sig = ar.alloc(sig_total + 1);
    for (int i = 0; i < njobs; i++) {
      if (m[i] < 0 || n[i] < 0 || l[i] < 0) throw Error(HM_EINVAL, "hm_test_trunc_batched: negative size");
      reqs[i] = TruncReq{m[i], n[i], l[i], a_dev + a_off[i], b_dev + b_off[i], ua_dev + o_off[i],
                         ub_dev + p_off[i], d_rank + i, d_sig + sig_off[i]};
    }
    trunc_batched(&ctx->c, ar, reqs, eps);
    HM_CUDA(cudaStreamSynchronize(ctx->c.stream));
    HM_CUDA(cudaMemcpy(ranks_host, d_rank, sizeof(int) * njobs, cudaMemcpyDeviceToHost));
    if (sigma_host) {
      std::vector<double> hs(sig_total + 1);
      HM_CUDA(cudaMemcpy(hs.data(), d_sig, sizeof(double) * (sig_total + 1), cudaMemcpyDeviceToHost));
      size_t o = 0;
      for (int i = 0; i < njobs; i++) {
        const int q = std::min(std::min(m[i], n[i]), l[i]);
        for (int j = 0; j < q; j++) sigma_host[o + j] = hs[sig_off[i] + j];
        o += q;
      }
    }
  });
}

hm_status hm_test_eval_batched(hm_ctx ctx, hm_mat H, int njobs, const int32_t* blk, const int32_t* trans,
                               const double* coef, double* v_dev, const int64_t* v_off, const int32_t* ldv,
                               double* out_dev, const int64_t* o_off, const int32_t* ldo, const int32_t* w,
                               double split_threshold) {
  if (!ctx || !H || njobs < 0 || (njobs > 0 && (!blk || !trans || !coef || !v_off || !ldv || !o_off || !ldo || !w)))
    return HM_EINVAL;
  return guard(ctx, [&] {
    set_device(ctx->c);
    std::vector<const double*> V(njobs);
    std::vector<double*> O(njobs);
    for (int i = 0; i < njobs; i++) {
      if (w[i] <= 0 || ldv[i] <= 0 || ldo[i] <= 0) throw Error(HM_EINVAL, "hm_test_eval_batched: bad panel shape");
      V[i] = v_dev + v_off[i];
      O[i] = out_dev + o_off[i];
    }
    eval_batched_test(&ctx->c, &H->m, njobs, blk, trans, coef, V.data(), ldv, O.data(), ldo, w, split_threshold);
  });
}

hm_status hm_flush_capture(hm_ctx ctx, uint64_t level_mask) {
  if (!ctx) return HM_EINVAL;
  return guard(ctx, [&] {
    set_device(ctx->c);
    ctx->c.cap_free();
    ctx->c.cap_on = true;
    ctx->c.cap_mask = level_mask;
  });
}

hm_status hm_flush_capture_info(hm_ctx ctx, int level, int64_t* njobs, int32_t* m, int32_t* n, int32_t* l,
                                int32_t* k, int* has_data) {
  if (!ctx || !njobs) return HM_EINVAL;
  return guard(ctx, [&] {
    if (level < 0) {            // number of captured levels
      *njobs = (int64_t)ctx->c.cap.size();
      return;
    }
    if (level >= (int)ctx->c.cap.size()) throw Error(HM_EINVAL, "hm_flush_capture_info: no such level");
    const Ctx::CapLevel& L = ctx->c.cap[level];
    *njobs = (int64_t)L.m.size();
    if (has_data) *has_data = L.data != nullptr;
    for (size_t i = 0; i < L.m.size(); i++) {
      if (m) m[i] = L.m[i];
      if (n) n[i] = L.n[i];
      if (l) l[i] = L.l[i];
      if (k) k[i] = i < L.k.size() ? L.k[i] : -1;
    }
  });
}

hm_status hm_flush_replay(hm_ctx ctx, int level, double eps, int reps, double* ms_out, int64_t* rank_sum) {
  if (!ctx) return HM_EINVAL;
  return guard(ctx, [&] {
    set_device(ctx->c);
    flush_replay(&ctx->c, level, eps, reps, ms_out, rank_sum);
  });
}

hm_status hm_flush_capture_free(hm_ctx ctx) {
  if (!ctx) return HM_EINVAL;
  return guard(ctx, [&] {
    set_device(ctx->c);
    ctx->c.cap_free();
    ctx->c.cap_on = false;
  });
}

}  // extern "C"
