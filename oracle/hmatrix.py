"""H-matrix container and basic operations (§2-3).

Representation (Def 2.4): admissible leaves hold (A_b, B_b)
with G|_b = A_b B_b^*, inadmissible leaves hold N_b = G|_b.  All data in
tree order (cluster index sets are contiguous ranges).

  build            dense leaves = exact entries; admissible leaves =
                   TRUNC_eps(G|_b): LAPACK gesvd if
                   min(m,n) <= 1024, else a randomized range finder
                   CERTIFIED by the directly computed residual
                   ||G_b - Q Q^T G_b||_F <= 1e-12 ||G_b||_F.
  addeval          Fig. 1, son ranges (SURVEY #3)
  addevaltrans     Fig. 1 with the typo fixed: X <- X + alpha N_b^* Y
  rkupdate         Fig. 3, N_b += alpha A B^* (alpha missing
                   at P:L464), restriction to t'x s'

Pinned by tests/test_oracle_hmatrix.py: exactness of addeval/addevaltrans
and rkupdate at eps = 0 against dense products, build at eps = 0 reproduces
the dense kernel matrix, build ranks/errors against per-block dense SVD,
certified randomized build equals LAPACK where both run.
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla

from . import kernel as K
from .lowrank import TruncCtx, choose_rank, trunc
from .trees import ADM, DENSE, SUB, build_block_tree, build_cluster_tree, tree_arrays


class HMatrix:
    """Leaf payloads over a (shared, immutable) block tree."""

    def __init__(self, bt):
        self.bt = bt
        self.A = {}   # block id -> (m x k)
        self.B = {}   # block id -> (n x k)
        self.N = {}   # block id -> (m x n)

    @property
    def n(self):
        return self.bt.rows.n

    def clone(self):
        h = HMatrix(self.bt)
        h.A = {k: v.copy() for k, v in self.A.items()}
        h.B = {k: v.copy() for k, v in self.B.items()}
        h.N = {k: v.copy() for k, v in self.N.items()}
        return h

    def rank(self, b):
        return self.A[b.id].shape[1]

    def ranks(self):
        return {bid: a.shape[1] for bid, a in self.A.items()}

    def to_dense(self, b=None):
        """Exact assembly of all leaves (test bridge)."""
        b = self.bt.root if b is None else b
        t0, s0 = b.t.start, b.s.start
        out = np.zeros((b.t.size, b.s.size))
        stack = [b]
        while stack:
            c = stack.pop()
            r = slice(c.t.start - t0, c.t.start - t0 + c.t.size)
            q = slice(c.s.start - s0, c.s.start - s0 + c.s.size)
            if c.kind == DENSE:
                out[r, q] = self.N[c.id]
            elif c.kind == ADM:
                out[r, q] = self.A[c.id] @ self.B[c.id].T
            else:
                stack.extend(c.sons)
        return out

    def storage(self):
        lr = sum(a.size + self.B[k].size for k, a in self.A.items())
        de = sum(v.size for v in self.N.values())
        return lr, de

    def set_zero(self):
        for b in self.bt.leaves():
            if b.kind == ADM:
                self.A[b.id] = np.zeros((b.t.size, 0))
                self.B[b.id] = np.zeros((b.s.size, 0))
            else:
                self.N[b.id] = np.zeros((b.t.size, b.s.size))


# ---------------------------------------------------------------- build

class Problem:
    """Trees + geometry of one configuration (no matrix data)."""

    def __init__(self, x, w, leaf_size, eta, kernel=K.KERNEL_SLP, nrm=None):
        self.x = np.asarray(x, np.float64)
        self.w = np.asarray(w, np.float64)
        self.nrm = None if nrm is None else np.asarray(nrm, np.float64)
        self.kernel = kernel
        self.ct = build_cluster_tree(self.x, leaf_size)
        self.bt = build_block_tree(self.ct, self.ct, eta)
        self.leaf_size = leaf_size
        self.eta = eta

    @property
    def perm(self):
        return self.ct.perm

    def block_entries(self, b):
        p = self.ct.perm
        return K.entries(self.x, self.w, p[b.t.start:b.t.start + b.t.size],
                         p[b.s.start:b.s.start + b.s.size], self.kernel, self.nrm)

    def dense(self):
        return K.dense_matrix(self.x, self.w, self.ct.perm, self.kernel, self.nrm)

    def arrays(self):
        return tree_arrays(self.ct, self.bt)


def _randomized_trunc(G, eps, seed, ctx_log=None):
    """SURVEY O3 large-block compression: randomized range finder with
    r = 64 columns, q = 2 power steps with re-orthonormalisation, certified by
    the DIRECT residual ||G - Q (Q^T G)||_F <= 1e-12 ||G||_F (never the
    Pythagoras difference); r doubles until certified.  Then exact SVD of
    Q^T G and the O4 rank rule."""
    m, n = G.shape
    gnorm = np.linalg.norm(G)
    r = 64
    while True:
        rng = np.random.default_rng([1703, 9085, 3, seed, r])
        Om = rng.standard_normal((n, min(r, n)))
        Q, _ = np.linalg.qr(G @ Om)
        for _ in range(2):
            Q, _ = np.linalg.qr(G.T @ Q)
            Q, _ = np.linalg.qr(G @ Q)
        W = Q.T @ G
        res = np.linalg.norm(G - Q @ W)
        if res <= 1e-12 * gnorm or r >= min(m, n):
            break
        r *= 2
    Uw, s, Vh = sla.svd(W, full_matrices=False, lapack_driver="gesvd")
    k, _ = choose_rank(s, eps)
    return Q @ Uw[:, :k], Vh[:k].T * s[:k], res / max(gnorm, 1e-300)


def build(prob: Problem, eps, ctx: TruncCtx | None = None):
    """hm_build: dense leaves exact; admissible leaves TRUNC_eps(G|_b)."""
    h = HMatrix(prob.bt)
    ctx = ctx or TruncCtx(eps, log_near=False)
    for b in prob.bt.leaves():
        G = prob.block_entries(b)
        if b.kind == DENSE:
            h.N[b.id] = G
            continue
        if min(G.shape) <= 1024:
            U, s, Vh = sla.svd(G, full_matrices=False, lapack_driver="gesvd")
            k, _ = choose_rank(s, eps)
            h.A[b.id] = U[:, :k].copy()
            h.B[b.id] = Vh[:k].T * s[:k]
        else:
            A, B, _ = _randomized_trunc(G, eps, b.id)
            h.A[b.id] = A
            h.B[b.id] = B
    return h


# ------------------------------------------------------ Fig. 1 addeval

def addeval(h: HMatrix, b, alpha, X, Y):
    """Y <- Y + alpha G|_{t x s} X  (Fig. 1); X: #s x c, Y: #t x c."""
    if b.kind == DENSE:
        Y += alpha * (h.N[b.id] @ X)
    elif b.kind == ADM:
        Zh = alpha * (h.B[b.id].T @ X)
        Y += h.A[b.id] @ Zh
    else:
        t0, s0 = b.t.start, b.s.start
        for c in b.sons:
            addeval(h, c, alpha,
                    X[c.s.start - s0:c.s.start - s0 + c.s.size],
                    Y[c.t.start - t0:c.t.start - t0 + c.t.size])


def addevaltrans(h: HMatrix, b, alpha, Y, X):
    """X <- X + alpha G|_{t x s}^* Y  (Fig. 1; P:L319 read as
    X <- X + alpha N_b^* Y); Y: #t x c, X: #s x c."""
    if b.kind == DENSE:
        X += alpha * (h.N[b.id].T @ Y)
    elif b.kind == ADM:
        Zh = alpha * (h.A[b.id].T @ Y)
        X += h.B[b.id] @ Zh
    else:
        t0, s0 = b.t.start, b.s.start
        for c in b.sons:
            addevaltrans(h, c, alpha,
                         Y[c.t.start - t0:c.t.start - t0 + c.t.size],
                         X[c.s.start - s0:c.s.start - s0 + c.s.size])


def matvec(h: HMatrix, alpha, X, Y, trans=False):
    b = h.bt.root
    if trans:
        addevaltrans(h, b, alpha, X, Y)
    else:
        addeval(h, b, alpha, X, Y)
    return Y


# ------------------------------------------------------ Fig. 3 rkupdate

def rkupdate(h: HMatrix, b, alpha, A, B, ctx: TruncCtx):
    """G|_{t x s} <- blocktrunc(G|_{t x s} + alpha A B^*)  (Fig. 3).
    A: #t x k, B: #s x k (restriction views by son offsets)."""
    if b.kind == DENSE:
        h.N[b.id] += alpha * (A @ B.T)
    elif b.kind == ADM:
        # rkadd(alpha, R, R')  (Fig. 2 stacking order [alpha A, C])
        h.A[b.id], h.B[b.id] = trunc(np.hstack([alpha * A, h.A[b.id]]),
                                     np.hstack([B, h.B[b.id]]), ctx)
    else:
        t0, s0 = b.t.start, b.s.start
        for c in b.sons:
            rkupdate(h, c, alpha,
                     A[c.t.start - t0:c.t.start - t0 + c.t.size],
                     B[c.s.start - s0:c.s.start - s0 + c.s.size], ctx)


# ------------------------------------------------------ export / import

def export(h: HMatrix, prob: Problem | None = None):
    """hm_host_desc schema (include/hm.h): tree arrays + per-block
    rank/offset + column-major factor and dense pools."""
    bt = h.bt
    d = tree_arrays(bt.rows, bt)
    nb = len(bt.blocks)
    rank = np.zeros(nb, np.int32)
    off = np.full(nb, -1, np.int64)
    fac, den = [], []
    fo = do = 0
    for b in bt.blocks:
        if b.kind == ADM:
            A, B = h.A[b.id], h.B[b.id]
            rank[b.id] = A.shape[1]
            off[b.id] = fo
            fac.append(A.ravel(order="F"))
            fac.append(B.ravel(order="F"))
            fo += A.size + B.size
        elif b.kind == DENSE:
            off[b.id] = do
            den.append(h.N[b.id].ravel(order="F"))
            do += h.N[b.id].size
    d["bl_rank"] = rank
    d["bl_off"] = off
    d["factors"] = np.concatenate(fac) if fac else np.zeros(0)
    d["dense"] = np.concatenate(den) if den else np.zeros(0)
    d["n"] = np.int64(bt.rows.n)
    return d


def import_payload(bt, d):
    """Inverse of export's payload part over an identical block tree."""
    h = HMatrix(bt)
    for b in bt.blocks:
        o = int(d["bl_off"][b.id])
        m, n = b.t.size, b.s.size
        if b.kind == ADM:
            k = int(d["bl_rank"][b.id])
            h.A[b.id] = d["factors"][o:o + m * k].reshape((m, k), order="F").copy()
            h.B[b.id] = d["factors"][o + m * k:o + (m + n) * k].reshape((n, k), order="F").copy()
        elif b.kind == DENSE:
            h.N[b.id] = d["dense"][o:o + m * n].reshape((m, n), order="F").copy()
    return h
