#!/usr/bin/env python3
"""Write oracle golden data for full-size parity tests (calls only oracle/ and
hm_inputs/; nothing from the CUDA path).

    python scripts/make_golden.py product 4     # BASELINE configs[3]: n=81920 product
    python scripts/make_golden.py lr 2          # configs[1]: n=5120 H-LR
    python scripts/make_golden.py chol 3        # configs[2]: n=20480 H-Cholesky

Stored in tests/golden/<name>.npz:
  ranks      per block rank of the result (-1 for non-admissible blocks)
  fro        per leaf block Frobenius norm of the result
  sample     ids of sampled leaf blocks; sketch_<id> = Z_b Omega_b with
             Omega_b = default_rng([1703, 9085, 99, id]).standard_normal((n_b, 4))
  probes     result applied to 2 probe vectors (tree order)
  meta       json (config, truncation counts, near-threshold list, timings)
"""
import json
import os
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

CONFIGS = {1: (3, 32, 1e-4), 2: (4, 32, 1e-4), 3: (5, 32, 1e-5), 4: (6, 64, 1e-6), 5: (7, 64, 1e-4)}


def omega(bid, n):
    return np.random.default_rng([1703, 9085, 99, int(bid)]).standard_normal((n, 4))


def summarise(P, H, nsample=400, max_rows=300):
    bt = P.bt
    nb = len(bt.blocks)
    ranks = np.full(nb, -1, np.int32)
    fro = np.zeros(nb)
    for b in bt.leaves():
        if b.kind == 1:
            A, B = H.A[b.id], H.B[b.id]
            ranks[b.id] = A.shape[1]
            _, Ra = np.linalg.qr(A)
            _, Rb = np.linalg.qr(B)
            fro[b.id] = np.linalg.norm(Ra @ Rb.T) if A.shape[1] else 0.0
        else:
            fro[b.id] = np.linalg.norm(H.N[b.id])
    rng = np.random.default_rng([1703, 9085, 98])
    cand = [b for b in bt.leaves() if b.t.size <= max_rows and b.s.size <= max_rows]
    pick = rng.choice(len(cand), size=min(nsample, len(cand)), replace=False)
    sample = np.array(sorted(cand[i].id for i in pick), np.int64)
    sk = {}
    for bid in sample:
        b = bt.blocks[bid]
        Om = omega(bid, b.s.size)
        if b.kind == 1:
            sk[f"sketch_{bid}"] = H.A[bid] @ (H.B[bid].T @ Om)
        else:
            sk[f"sketch_{bid}"] = H.N[bid] @ Om
    return ranks, fro, sample, sk


def main():
    what, cfg = sys.argv[1], int(sys.argv[2])
    workers = int(sys.argv[3]) if len(sys.argv) > 3 else os.cpu_count()
    L, leaf, eps = CONFIGS[cfg]
    x, w = sphere_points(L)
    kernel = K.KERNEL_SLP_SYM if what == "chol" else K.KERNEL_SLP
    P = Problem(x, w, leaf, 2.0, kernel=kernel)
    t0 = time.time()
    G = build_parallel(P, eps, workers)
    t_build = time.time() - t0
    print(f"build n={P.ct.n}: {t_build:.1f}s", flush=True)
    meta = dict(what=what, config=cfg, L=L, leaf=leaf, eps=eps, n=int(P.ct.n), build_s=t_build)
    t0 = time.time()
    if what == "product":
        Z, info = addmul_s2_parallel(1.0, G.clone(), G.clone(), G.clone(), eps, workers)
        meta.update({k: (v if k != "near" else [list(map(str, x)) for x in v]) for k, v in info.items()})
        out = Z
    else:
        from oracle.factor import chol_with_restart, lr, probe_residual
        from oracle.lowrank import TruncCtx
        ctx = TruncCtx(eps)
        G0 = G.clone()
        if what == "lr":
            out, F = lr(G, eps, ctx=ctx)
            shift = 0.0
        else:
            out, F, shift = chol_with_restart(G, eps, lambda: TruncCtx(eps))
            ctx = F.ctx
        v = probe_vectors(P.ct.n)[P.perm]
        meta.update(truncations=ctx.count, trunc_cols=ctx.cols, near=[str(x[1]) for x in ctx.near],
                    min_pivot=F.min_pivot, shift=shift,
                    probe_residual=probe_residual(G0, out, v, what, shift))
    meta["op_s"] = time.time() - t0
    print(f"{what}: {meta['op_s']:.1f}s truncations {meta['truncations']}", flush=True)
    ranks, fro, sample, sk = summarise(P, out)
    v = probe_vectors(P.ct.n, 2)[P.perm]
    pr = np.zeros_like(v)
    matvec(out, 1.0, v, pr)
    os.makedirs(os.path.join(ROOT, "tests", "golden"), exist_ok=True)
    path = os.path.join(ROOT, "tests", "golden", f"{what}_cfg{cfg}.npz")
    np.savez_compressed(path, ranks=ranks, fro=fro, sample=sample, probes=pr, meta=json.dumps(meta), **sk)
    print("wrote", path, os.path.getsize(path) // 1024, "KiB", flush=True)


if __name__ == "__main__":
    main()
