#!/usr/bin/env python3
"""Write oracle golden data for full-size parity tests (calls only oracle/ and
hm_inputs/; nothing from the CUDA path).

    python scripts/make_golden.py product 1     # BASELINE configs[0]: n=1280 product
    python scripts/make_golden.py product 4     # configs[3]: n=81920 product
    python scripts/make_golden.py lr 2          # configs[1]: n=5120 H-LR
    python scripts/make_golden.py chol 3        # configs[2]: n=20480 H-Cholesky
    python scripts/make_golden.py lr 4          # "config 4'": H-LR of configs[3]'s matrix (metric, n=81920)
    python scripts/make_golden.py lr 5          # configs[4]: n=327680 H-LR
    [workers]  (default: all host cores)

The built H-matrix and the oracle's result are also pickled under
.golden_raw/ (git- and gpurun-ignored) so summaries can be recomputed and
config 4 / 4' share one build.

tests/golden/<what>_cfg<cfg>.npz (oracle/summary.py):
  leaf_ids, ranks, fro, sk     summary of the RESULT for every leaf block:
                               rank, exact ||Z_b||_F, two-sided sketch
                               Omega_L[t]^T Z_b Omega_R[r] (sketch_k x sketch_k)
  b_ranks, b_fro               summary of the BUILT input (build parity)
  probes                       result applied to 2 probe vectors (tree order;
                               H-LR: L(R v), Cholesky: L(L^T v))
  near                         (t, r) cluster ids of near-threshold truncations
  meta                         json: config, truncation counts, timings
"""
import json
import os
import pickle
import sys
import time

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from hm_inputs import probe_vectors, sphere_points  # noqa: E402
from oracle import kernel as K  # noqa: E402
from oracle.hmatrix import Problem, matvec  # noqa: E402
from oracle.parallel import addmul_s2_parallel, build_parallel  # noqa: E402
from oracle.summary import summarise_hmatrix  # noqa: E402

# cfg -> (icosphere level, leaf, eps); BASELINE.json configs[cfg-1]; 4 = configs[3]'s matrix
CONFIGS = {1: (3, 32, 1e-4), 2: (4, 32, 1e-4), 3: (5, 32, 1e-5), 4: (6, 64, 1e-6), 5: (7, 64, 1e-4)}
RAW = os.path.join(ROOT, ".golden_raw")


def near_tags(near):
    """(t, r) cluster ids of near-threshold truncations; tags are
    (kind, t_id, r_id) (oracle/product.py, oracle/factor.py)."""
    out = []
    for tag in near:
        if tag is not None and len(tag) >= 3:
            out.append((int(tag[1]), int(tag[2])))
    return sorted(set(out))


def get_build(P, eps, kernel, L, leaf, workers):
    os.makedirs(RAW, exist_ok=True)
    path = os.path.join(RAW, f"build_L{L}_leaf{leaf}_eps{eps:g}_k{kernel}.pkl")
    if os.path.exists(path):
        with open(path, "rb") as f:
            G, t_build = pickle.load(f)
        print(f"build loaded from {path}", flush=True)
        return G, t_build
    t0 = time.time()
    G = build_parallel(P, eps, workers)
    t_build = time.time() - t0
    with open(path, "wb") as f:
        pickle.dump((G, t_build), f, protocol=pickle.HIGHEST_PROTOCOL)
    return G, t_build


def main():
    what, cfg = sys.argv[1], int(sys.argv[2])
    workers = int(sys.argv[3]) if len(sys.argv) > 3 else os.cpu_count()
    L, leaf, eps = CONFIGS[cfg]
    x, w = sphere_points(L)
    kernel = K.KERNEL_SLP_SYM if what == "chol" else K.KERNEL_SLP
    P = Problem(x, w, leaf, 2.0, kernel=kernel)
    G, t_build = get_build(P, eps, kernel, L, leaf, workers)
    print(f"build n={P.ct.n}: {t_build:.1f}s", flush=True)
    meta = dict(what=what, config=cfg, L=L, leaf=leaf, eps=eps, n=int(P.ct.n), kernel=kernel, build_s=t_build)
    sk_k = 2 if cfg == 5 else 4
    bsum = summarise_hmatrix(G, sk_k)
    t0 = time.time()
    v2 = probe_vectors(P.ct.n, 2)[P.perm]
    if what == "product":
        Z, info = addmul_s2_parallel(1.0, G.clone(), G.clone(), G.clone(), eps, workers, frontier_depth=4)
        near = near_tags(t for t, _ in info["near"])
        meta.update(truncations=info["truncations"], trunc_cols=info["trunc_cols"],
                    addproduct=info["addproduct"], frontier=info["frontier"], schedule="S2 (oracle.parallel)")
        out = Z
        meta["op_s"] = time.time() - t0
        pr = np.zeros_like(v2)
        matvec(out, 1.0, v2, pr)
    else:
        from oracle.factor import apply_factor, chol_with_restart, lr, probe_residual
        from oracle.lowrank import TruncCtx
        ctx = TruncCtx(eps)
        G0 = G.clone()
        Gw = G.clone()
        if what == "lr":
            out, F = lr(Gw, eps, ctx=ctx)
            shift = 0.0
        else:
            out, F, shift = chol_with_restart(Gw, eps, lambda: TruncCtx(eps))
            ctx = F.ctx
        meta["op_s"] = time.time() - t0
        near = near_tags(x[1] for x in ctx.near)
        v8 = probe_vectors(P.ct.n)[P.perm]
        meta.update(truncations=ctx.count, trunc_cols=ctx.cols, min_pivot=F.min_pivot, shift=shift,
                    probe_residual=probe_residual(G0, out, v8, what, shift), schedule="O8/O9 (oracle.factor)")
        if what == "lr":
            pr = apply_factor(out, "L", apply_factor(out, "R", v2))
        else:
            pr = apply_factor(out, "Lc", apply_factor(out, "LcT", v2))
    meta["near_count"] = len(near)
    print(f"{what} cfg{cfg}: {meta['op_s']:.1f}s truncations {meta['truncations']} near {len(near)}", flush=True)
    with open(os.path.join(RAW, f"{what}_cfg{cfg}_result.pkl"), "wb") as f:
        pickle.dump((out, meta, near), f, protocol=pickle.HIGHEST_PROTOCOL)
    rsum = summarise_hmatrix(out, sk_k)
    os.makedirs(os.path.join(ROOT, "tests", "golden"), exist_ok=True)
    path = os.path.join(ROOT, "tests", "golden", f"{what}_cfg{cfg}.npz")
    np.savez_compressed(path, leaf_ids=rsum["leaf_ids"], ranks=rsum["ranks"], fro=rsum["fro"], sk=rsum["sk"],
                        b_ranks=bsum["ranks"], b_fro=bsum["fro"], probes=pr,
                        near=np.array(near, np.int64).reshape(-1, 2), meta=json.dumps(meta))
    print("wrote", path, os.path.getsize(path) // 1024, "KiB", flush=True)


if __name__ == "__main__":
    main()
