"""Process-parallel drivers of the oracle (test infrastructure / CPU baseline).

The Parallelization remark says flushes of different sons are
independent; the oracle uses that to run large configurations on all host
cores.  The arithmetic is exactly the serial oracle's (same functions, same
order inside every subtree), so results are identical to the serial runs:
  * build_parallel: admissible blocks compressed by independent workers
    (OPENBLAS_NUM_THREADS=1 each);
  * addmul_s2_parallel: the S2 product is run serially down to a frontier of
    independent (accumulator, Z block) pairs, whose flushes run in workers
    (fork: X, Y, Z shared copy-on-write); workers return their Z leaves.
"""
from __future__ import annotations

import multiprocessing as mp
import os

import numpy as np

from .hmatrix import HMatrix, build
from .lowrank import TruncCtx, choose_rank
from .product import S2, Acc2, Stats, ZReal
from .trees import ADM, DENSE, SUB

_G = {}


def _build_worker(ids):
    import scipy.linalg as sla
    from .hmatrix import _randomized_trunc
    prob, eps = _G["prob"], _G["eps"]
    out = {}
    for bid in ids:
        b = prob.bt.blocks[bid]
        G = prob.block_entries(b)
        if min(G.shape) <= 1024:
            U, s, Vh = sla.svd(G, full_matrices=False, lapack_driver="gesvd")
            k, _ = choose_rank(s, eps)
            out[bid] = (U[:, :k].copy(), Vh[:k].T * s[:k])
        else:
            A, B, _ = _randomized_trunc(G, eps, b.id)
            out[bid] = (A, B)
    return out


def build_parallel(prob, eps, workers=None):
    workers = workers or os.cpu_count()
    h = HMatrix(prob.bt)
    adm = []
    for b in prob.bt.leaves():
        if b.kind == DENSE:
            h.N[b.id] = prob.block_entries(b)
        else:
            adm.append(b)
    adm.sort(key=lambda b: -b.t.size * b.s.size)
    chunks = [[] for _ in range(workers * 4)]
    for i, b in enumerate(adm):   # round robin over size-sorted blocks (load balance)
        chunks[i % len(chunks)].append(b.id)
    _G.update(prob=prob, eps=eps)
    with mp.get_context("fork").Pool(workers) as pool:
        for res in pool.imap_unordered(_build_worker, chunks):
            for bid, (A, B) in res.items():
                h.A[bid], h.B[bid] = A, B
    return h


def _subtree_leaves(b):
    out, st = [], [b]
    while st:
        x = st.pop()
        if x.kind == SUB:
            st.extend(x.sons)
        else:
            out.append(x)
    return out


def _flush_worker(i):
    acc, zb = _G["items"][i]
    X, Y, Z, eps = _G["X"], _G["Y"], _G["Z"], _G["eps"]
    from .flops import ConventionCounter
    ctx = TruncCtx(eps)
    cc = ConventionCounter()
    alg = S2(X, Y, ctx, Stats(), counter=cc)
    b = Z.bt.blocks[zb]
    alg.flush(acc, ZReal(Z, b))
    out = {}
    for leaf in _subtree_leaves(b):
        if leaf.kind == ADM:
            out[leaf.id] = ("A", Z.A[leaf.id], Z.B[leaf.id])
        else:
            out[leaf.id] = ("N", Z.N[leaf.id])
    return i, out, ctx.count, ctx.cols, [(n[1], n[2]) for n in ctx.near], alg.st.addproduct, cc.total_flops()


def addmul_s2_parallel(alpha, X: HMatrix, Y: HMatrix, Z: HMatrix, eps, workers=None, frontier_depth=3):
    """Z <- blocktrunc(Z + alpha X Y), S2 schedule, identical to addmul_s2."""
    from .flops import ConventionCounter
    workers = workers or os.cpu_count()
    ctx = TruncCtx(eps)
    cc = ConventionCounter()   # SURVEY §8(d) convention work (timing reports only)
    alg = S2(X, Y, ctx, Stats(), counter=cc)
    root = Z.bt.root
    acc = Acc2(root.t, root.s)
    alg.addproduct(acc, alpha, X.bt.root, Y.bt.root)
    items = []

    def descend(a, z, d):
        if d == 0 or not a.pending or z.kind != SUB:
            items.append((a, z.b.id))
            return
        grid = alg.split(a, (z.t.id, z.r.id))
        for i in range(len(grid)):
            for j in range(len(grid[i])):
                descend(grid[i][j], z.son(i, j), d - 1)

    descend(acc, ZReal(Z, root), frontier_depth)
    _G.update(items=items, X=X, Y=Y, Z=Z, eps=eps)
    count, cols, near, addp = ctx.count, ctx.cols, [(n[1], n[2]) for n in ctx.near], alg.st.addproduct
    with mp.get_context("fork").Pool(workers) as pool:
        conv = cc.total_flops()
        for i, out, c, l, nr, ap, fl in pool.imap_unordered(_flush_worker, range(len(items))):
            conv += fl
            for bid, v in out.items():
                if v[0] == "A":
                    Z.A[bid], Z.B[bid] = v[1], v[2]
                else:
                    Z.N[bid] = v[1]
            count += c
            cols += l
            near += nr
            addp += ap
    # near: (tag, k) of every near-threshold truncation (tags carry the (t, r) cluster ids)
    return Z, dict(truncations=count, trunc_cols=cols, near=near, addproduct=addp, frontier=len(items),
                   conv_gflop=conv / 1e9)
