"""H-matrix inversion with accumulated updates (§6, Fig. 8,
P:L1441-1535) -- TEST INFRASTRUCTURE (see oracle/__init__.py).

invert(t, acc): G|tt + content(acc) is replaced by its inverse, in place,
following Fig. 8 line by line (block LR factorization of G|tt, six steps
P:L1441-1450), with the S2 accumulators of oracle/product.py:

    leaf t:  flush(acc -> G_tt) (Fig. 7 ii); G_tt <- G_tt^{-1} (dense, LAPACK)
    else:    split(acc) -> acc_11, acc_12, acc_21, acc_22          (Fig. 6, T1)
             invert(t1, acc_11)                                    G11 <- G11^{-1}
             flush(acc_12 -> G12); flush(acc_21 -> G21)
             H12 <- 0; H21 <- 0
             addproduct(1, G11, G12 -> acc_12); flush(acc_12 -> H12)   H12 = G11^{-1} G12
             addproduct(1, G21, G11 -> acc_21); flush(acc_21 -> H21)   H21 = G21 G11^{-1}
             addproduct(-1, H21, G12 -> acc_22)                        S = G22 - H21 G12 (pending)
             invert(t2, acc_22)                                        G22 <- S^{-1}
             G12 <- 0; G21 <- 0
             addproduct(-1, H12, G22 -> acc_12); flush(acc_12 -> G12)  G12 = -H12 S^{-1}
             addproduct(-1, G22, H21 -> acc_21); flush(acc_21 -> G21)  G21 = -S^{-1} H21
             addproduct(-1, H12, G21 -> acc_11); flush(acc_11 -> G11)  G11 = G11^{-1} + H12 S^{-1} H21

Readings:
  * R21 = SURVEY ambiguity #6: Fig. 8's last addproduct is printed into
    R_hat_{t2,t2} but flushed into G11: it must be the
    accumulator of (t1, t1) -- the block it is flushed into.
  * The auxiliary H is an H-matrix over the same block tree; only its blocks
    (t1,t2) / (t2,t1) of the current recursion level are used.
  * "flush" into a subdivided block with no pending products is Fig. 7's
    branch (iii) (reduce, then every leaf gets T2 / an exact add).
  * Dense leaf inverse: numpy.linalg.inv (LAPACK getrf/getri; the paper's
    "standard linear algebra").

Pinned by tests/test_oracle_inverse.py: at eps = 0 on tiny n the result is
the exact inverse (G G^{-1} = I to 1e-10 against the dense matrix); a
block-diagonal input inverts blockwise; the preconditioner error
||I - G~^{-1} G||_2 at eps = 1e-4 stays within the eps-scaled range the
paper reports."""
from __future__ import annotations

import numpy as np

from .hmatrix import HMatrix
from .lowrank import TruncCtx
from .product import S2, Acc2, Stats, ZReal
from .trees import ADM, DENSE, SUB


def _zero_subtree(h: HMatrix, b):
    st = [b]
    while st:
        x = st.pop()
        if x.kind == SUB:
            st.extend(x.sons)
        elif x.kind == ADM:
            h.A[x.id] = np.zeros((x.t.size, 0))
            h.B[x.id] = np.zeros((x.s.size, 0))
        else:
            h.N[x.id] = np.zeros((x.t.size, x.s.size))


class Inverter:
    def __init__(self, G: HMatrix, eps, ctx: TruncCtx | None = None):
        self.G = G
        self.H = HMatrix(G.bt)
        self.H.set_zero()
        self.ctx = ctx or TruncCtx(eps)
        self.alg = S2(G, G, self.ctx, Stats())
        self.leaf_inverses = 0

    def flush(self, acc, h, b):
        self.alg.flush(acc, ZReal(h, b))

    def invert(self, t, acc):
        G, H, alg = self.G, self.H, self.alg
        find = G.bt.find
        if t.leaf:
            b = find(t, t)
            self.flush(acc, G, b)
            G.N[b.id] = np.linalg.inv(G.N[b.id])
            self.leaf_inverses += 1
            return
        grid = alg.split(acc, (t.id, t.id))
        t1, t2 = t.sons
        b11, b12, b21, b22 = find(t1, t1), find(t1, t2), find(t2, t1), find(t2, t2)
        self.invert(t1, grid[0][0])
        self.flush(grid[0][1], G, b12)
        self.flush(grid[1][0], G, b21)
        _zero_subtree(H, b12)
        _zero_subtree(H, b21)
        a12 = Acc2(t1, t2)
        alg.addproduct(a12, 1.0, b11, b12, G, G)
        self.flush(a12, H, b12)                        # H12 = G11^{-1} G12
        a21 = Acc2(t2, t1)
        alg.addproduct(a21, 1.0, b21, b11, G, G)
        self.flush(a21, H, b21)                        # H21 = G21 G11^{-1}
        alg.addproduct(grid[1][1], -1.0, b21, b12, H, G)   # S = G22 - H21 G12
        self.invert(t2, grid[1][1])                    # G22 <- S^{-1}
        _zero_subtree(G, b12)
        _zero_subtree(G, b21)
        a12 = Acc2(t1, t2)
        alg.addproduct(a12, -1.0, b12, b22, H, G)
        self.flush(a12, G, b12)                        # G12 = -H12 S^{-1}
        a21 = Acc2(t2, t1)
        alg.addproduct(a21, -1.0, b22, b21, G, H)
        self.flush(a21, G, b21)                        # G21 = -S^{-1} H21
        a11 = Acc2(t1, t1)                             # reading R21: acc_(t1,t1)
        alg.addproduct(a11, -1.0, b12, b21, H, G)
        self.flush(a11, G, b11)                        # G11 = G11^{-1} - H12 G21


def _check_binary(G):
    for c in G.bt.rows.clusters:
        if c.sons and len(c.sons) != 2:
            raise ValueError("inversion needs a binary cluster tree (P:L1361-1363)")


def invert(G: HMatrix, eps, ctx=None):
    """In place: G <- approximate G^{-1} (Fig. 8 with accumulators)."""
    _check_binary(G)
    inv = Inverter(G, eps, ctx)
    root = G.bt.root
    inv.invert(root.t, Acc2(root.t, root.s))
    return G, inv


def inverse_precond_error(G0: HMatrix, Ginv: HMatrix, iters=30, seed=0):
    """||I - G~^{-1} G||_2 by power iteration on E^T E,
    E = I - Ginv G0 (both applied by addeval, Fig. 1)."""
    from .hmatrix import matvec
    n = G0.n
    v = np.random.default_rng([1703, 9085, 6, seed]).standard_normal(n)
    v /= np.linalg.norm(v)
    est = 0.0
    for _ in range(iters):
        gv = np.zeros(n)
        matvec(G0, 1.0, v, gv)
        y = np.zeros(n)
        matvec(Ginv, 1.0, gv, y)
        w = v - y
        est = float(np.linalg.norm(w))
        z1 = np.zeros(n)
        matvec(Ginv, 1.0, w, z1, trans=True)
        z = np.zeros(n)
        matvec(G0, 1.0, z1, z, trans=True)
        u = w - z
        nu = np.linalg.norm(u)
        if nu == 0.0:
            return 0.0
        v = u / nu
    return est
