"""H-LR and H-Cholesky factorizations with accumulated updates (§6).

The paper states only that "the same holds for the H-LR and the H-Cholesky
factorizations" and runs them in §7; the
recursions are not printed.  Readings:

  LR(t, acc):  G|tt + content(acc) = L_tt R_tt, in place (strict lower = L,
      unit diagonal implicit; upper incl. diagonal = R)
    leaf t:  flush(acc -> G_tt) (Fig. 7 branch ii), dense LU without pivoting
    else:    split(acc) (Fig. 6, T1 reduce) -> acc_11, acc_12, acc_21, acc_22
             LR(t1, acc_11)
             SOLVE_L(t1, (t1,t2), acc_12)      R_12 = L_11^-1 (G_12 + content)
             SOLVE_R(t1, (t2,t1), acc_21)      L_21 = (G_21 + content) R_11^-1
             addproduct(-1, t1, L_21, R_12 -> acc_22)   (Fig. 5)
             LR(t2, acc_22)
  SOLVE_L(t, b, acc): admissible/dense leaf: flush, then the exact triangular
      solve of the factor A_b / the panel N_b (TRSM_L through the H-structure,
      addeval with alpha = -1, Fig. 1); subdivided: split, then for every
      column son r': SOLVE_L(t1), addproduct(-1, t1, L_(t2,t1), R_(t1,r')),
      SOLVE_L(t2).  SOLVE_R is the transpose.
  The accumulator is passed down and flushed only into a leaf that becomes a
  factorization or solve target (the accumulator analogue of Fig. 8's flush
  discipline).

  CHOL(t, acc): the same on the lower triangle: split makes only lower sons,
      SOLVE_LT(t1, (t2,t1)) gives L_21 = (G_21 + content) L_11^-T, and
      addproduct(-1, t1, L_21, L_21^T -> acc_22) uses a transpose view.

Dense leaf LU: no pivoting, unit L; |pivot| <= 1e-300 or non-finite raises
PivotError naming the cluster.  Cholesky: numpy on the lower triangle.

Pinned by tests/test_oracle_factor.py: eps = 0 on tiny n gives L R = G and
L L^T = G to 1e-10 (dense oracle); block-diagonal input gives blockwise
factors; leaf LU equals scipy.linalg.lu when its permutation is I; probe
residuals of the configs below 50 eps (SURVEY #21).
"""
from __future__ import annotations

from collections.abc import Mapping

import numpy as np
import scipy.linalg as sla

from .hmatrix import HMatrix, addeval, addevaltrans
from .lowrank import TruncCtx
from .product import S2, Acc2, Stats, ZReal
from .trees import ADM, DENSE, SUB


class PivotError(ArithmeticError):
    def __init__(self, cluster, value):
        super().__init__(f"pivot breakdown in leaf cluster {cluster.id} "
                         f"[{cluster.start}:{cluster.start + cluster.size}] (pivot {value!r})")
        self.cluster = cluster
        self.value = value


# ------------------------------------------------------------ dense leaves

def lu_nopivot(N, cluster=None):
    """In-place right-looking LU without pivoting: N = L R, unit lower L."""
    n = N.shape[0]
    for j in range(n):
        piv = N[j, j]
        if not np.isfinite(piv) or abs(piv) <= 1e-300:
            raise PivotError(cluster, piv)
        N[j + 1:, j] /= piv
        N[j + 1:, j + 1:] -= np.outer(N[j + 1:, j], N[j, j + 1:])
    return N


def chol_lower(N, cluster=None):
    try:
        L = np.linalg.cholesky(N)          # reads the lower triangle
    except np.linalg.LinAlgError:
        raise PivotError(cluster, float(np.min(np.diag(N))))
    N[:] = L
    return N


# ------------------------------------------------------------ transpose view

class _TMap(Mapping):
    def __init__(self, src, tmap, transpose):
        self.src, self.tmap, self.t = src, tmap, transpose

    def __getitem__(self, k):
        v = self.src[self.tmap[k]]
        return v.T if self.t else v

    def __iter__(self):
        return iter(self.tmap)

    def __len__(self):
        return len(self.tmap)


class TransposeView:
    """H-matrix view of G^T over the same (symmetric) block tree:
    block (s,r) of the view is block (r,s) of G, transposed."""

    def __init__(self, h: HMatrix):
        bt = h.bt
        self.bt = bt
        tmap = {}
        for b in bt.blocks:
            tb = bt.find(b.s, b.t)
            if tb is None or tb.kind != b.kind:
                raise ValueError("transpose view needs a symmetric block tree")
            tmap[b.id] = tb.id
        self.A = _TMap(h.B, {k: v for k, v in tmap.items() if bt.blocks[k].kind == ADM}, False)
        self.B = _TMap(h.A, {k: v for k, v in tmap.items() if bt.blocks[k].kind == ADM}, False)
        self.N = _TMap(h.N, {k: v for k, v in tmap.items() if bt.blocks[k].kind == DENSE}, True)


# ------------------------------------------------------------ helpers

def _diag(h, t):
    return h.bt.find(t, t)


def _rows(parent, son):
    return slice(son.start - parent.start, son.start - parent.start + son.size)


def is_lower(b):
    return b.t.start >= b.s.start


class Factorizer:
    """Shared machinery: S2 accumulators (oracle/product.py) on G in place."""

    def __init__(self, G: HMatrix, eps, ctx: TruncCtx | None = None, cholesky=False):
        self.G = G
        self.eps = eps
        self.ctx = ctx or TruncCtx(eps)
        self.chol = cholesky
        self.Y = TransposeView(G) if cholesky else G
        self.alg = S2(G, self.Y, self.ctx, Stats())
        self.min_pivot = np.inf

    # ---- triangular solves with H-matrix triangular factors (exact)
    def trsm_l(self, t, V, unit):
        """V <- L_tt^{-1} V (lower triangle of the diagonal blocks of G)."""
        if t.leaf:
            N = self.G.N[_diag(self.G, t).id]
            V[:] = sla.solve_triangular(N, V, lower=True, unit_diagonal=unit)
            return
        t1, t2 = t.sons
        self.trsm_l(t1, V[_rows(t, t1)], unit)
        addeval(self.G, self.G.bt.find(t2, t1), -1.0, V[_rows(t, t1)], V[_rows(t, t2)])
        self.trsm_l(t2, V[_rows(t, t2)], unit)

    def trsm_rt(self, s, V):
        """V <- R_ss^{-T} V (upper triangle of G incl. diagonal)."""
        if s.leaf:
            N = self.G.N[_diag(self.G, s).id]
            V[:] = sla.solve_triangular(N, V, lower=False, trans="T")
            return
        s1, s2 = s.sons
        self.trsm_rt(s1, V[_rows(s, s1)])
        addevaltrans(self.G, self.G.bt.find(s1, s2), -1.0, V[_rows(s, s1)], V[_rows(s, s2)])
        self.trsm_rt(s2, V[_rows(s, s2)])

    def flush_leaf(self, acc, b):
        self.alg.flush(acc, ZReal(self.G, b))

    # ---- LR (O8)
    def lr(self, t, acc):
        G = self.G
        if t.leaf:
            b = _diag(G, t)
            self.flush_leaf(acc, b)
            N = G.N[b.id]
            lu_nopivot(N, t)
            self.min_pivot = min(self.min_pivot, float(np.min(np.abs(np.diag(N)))))
            return
        grid = self.alg.split(acc, (t.id, t.id))
        t1, t2 = t.sons
        self.lr(t1, grid[0][0])
        self.solve_l(t1, G.bt.find(t1, t2), grid[0][1])
        self.solve_r(t1, G.bt.find(t2, t1), grid[1][0])
        self.alg.addproduct(grid[1][1], -1.0, G.bt.find(t2, t1), G.bt.find(t1, t2))
        self.lr(t2, grid[1][1])

    def solve_l(self, t, b, acc, unit=True):
        """G_b <- L_tt^{-1} (G_b + content(acc)), b = (t, r)."""
        G = self.G
        if b.kind == ADM:
            self.flush_leaf(acc, b)
            self.trsm_l(t, G.A[b.id], unit)
        elif b.kind == DENSE:
            self.flush_leaf(acc, b)
            self.trsm_l(t, G.N[b.id], unit)
        else:
            grid = self.alg.split(acc, (b.t.id, b.s.id))
            t1, t2 = b.t.sons
            for j, rj in enumerate(b.s.sons):
                self.solve_l(t1, G.bt.find(t1, rj), grid[0][j], unit)
                self.alg.addproduct(grid[1][j], -1.0, G.bt.find(t2, t1), G.bt.find(t1, rj))
                self.solve_l(t2, G.bt.find(t2, rj), grid[1][j], unit)

    def solve_r(self, s, b, acc):
        """G_b <- (G_b + content(acc)) R_ss^{-1}, b = (t, s)."""
        G = self.G
        if b.kind == ADM:
            self.flush_leaf(acc, b)
            self.trsm_rt(s, G.B[b.id])
        elif b.kind == DENSE:
            self.flush_leaf(acc, b)
            NT = G.N[b.id].T.copy()
            self.trsm_rt(s, NT)
            G.N[b.id][:] = NT.T
        else:
            grid = self.alg.split(acc, (b.t.id, b.s.id))
            s1, s2 = b.s.sons
            for i, ti in enumerate(b.t.sons):
                self.solve_r(s1, G.bt.find(ti, s1), grid[i][0])
                self.alg.addproduct(grid[i][1], -1.0, G.bt.find(ti, s1), G.bt.find(s1, s2))
                self.solve_r(s2, G.bt.find(ti, s2), grid[i][1])

    # ---- Cholesky (O9)
    def cholesky(self, t, acc):
        G = self.G
        if t.leaf:
            b = _diag(G, t)
            self.flush_leaf(acc, b)
            N = G.N[b.id]
            chol_lower(N, t)
            N[np.triu_indices(N.shape[0], 1)] = 0.0
            self.min_pivot = min(self.min_pivot, float(np.min(np.diag(N))))
            return
        grid = self.alg.split(acc, (t.id, t.id), lower_only=True)
        t1, t2 = t.sons
        self.cholesky(t1, grid[0][0])
        self.solve_lt(t1, G.bt.find(t2, t1), grid[1][0])
        self.alg.addproduct(grid[1][1], -1.0, G.bt.find(t2, t1), G.bt.find(t1, t2))   # Y = L^T view
        self.cholesky(t2, grid[1][1])

    def trsm_lnu(self, s, V):
        """V <- L_ss^{-1} V with the (non-unit) Cholesky factor."""
        self.trsm_l(s, V, unit=False)

    def solve_lt(self, s, b, acc):
        """G_b <- (G_b + content(acc)) L_ss^{-T}, b = (t, s) strictly lower."""
        G = self.G
        if b.kind == ADM:
            self.flush_leaf(acc, b)
            self.trsm_lnu(s, G.B[b.id])
        elif b.kind == DENSE:
            self.flush_leaf(acc, b)
            NT = G.N[b.id].T.copy()
            self.trsm_lnu(s, NT)
            G.N[b.id][:] = NT.T
        else:
            grid = self.alg.split(acc, (b.t.id, b.s.id))
            s1, s2 = b.s.sons
            for i, ti in enumerate(b.t.sons):
                self.solve_lt(s1, G.bt.find(ti, s1), grid[i][0])
                self.alg.addproduct(grid[i][1], -1.0, G.bt.find(ti, s1), G.bt.find(s1, s2))  # L^T view
                self.solve_lt(s2, G.bt.find(ti, s2), grid[i][1])


def _check_binary(G):
    for c in G.bt.rows.clusters:
        if c.sons and len(c.sons) != 2:
            raise ValueError("H-LR/H-Cholesky need a binary cluster tree (P:L1361-1363)")


def lr(G: HMatrix, eps, ctx=None):
    """In place: strict lower part = L (unit diagonal), upper part = R."""
    _check_binary(G)
    F = Factorizer(G, eps, ctx)
    root = G.bt.root
    F.lr(root.t, Acc2(root.t, root.s))
    return G, F


def chol(G: HMatrix, eps, shift=0.0, ctx=None):
    """In place lower L with L L^T = G + shift I (upper blocks untouched)."""
    _check_binary(G)
    if shift:
        for b in G.bt.leaves():
            if b.t is b.s:
                G.N[b.id][np.diag_indices(b.t.size)] += shift
    F = Factorizer(G, eps, ctx, cholesky=True)
    root = G.bt.root
    F.cholesky(root.t, Acc2(root.t, root.s))
    return G, F


def chol_with_restart(G: HMatrix, eps, ctx_factory=None):
    """SURVEY O9 / BASELINE config 3: on pivot failure restart the whole
    factorization with G + delta I, delta = 1e-6 max |G_ii|; returns (L, F, delta)."""
    G0 = G.clone()
    try:
        L, F = chol(G, eps, 0.0, ctx_factory() if ctx_factory else None)
        return L, F, 0.0
    except PivotError:
        dmax = max(float(np.max(np.abs(np.diag(G0.N[b.id])))) for b in G0.bt.leaves() if b.t is b.s)
        delta = 1e-6 * dmax
        L, F = chol(G0, eps, delta, ctx_factory() if ctx_factory else None)
        return L, F, delta


# ------------------------------------------------------------ applying factors

def apply_factor(F: HMatrix, part, V):
    """Y = op(F) V for part in {'L' (unit lower), 'R' (upper), 'Lc' (lower, non-unit),
    'LcT' (transpose of Lc), 'LT' (transpose of L), 'RT' (transpose of R)} using
    the leaves of the in-place factorization."""
    if part in ("LT", "RT"):
        # op(F)^T V = (op(F)^T applied by rows): Y = (M^T) V with M = apply_factor(part[0])
        base = part[0]
        Y = np.zeros_like(V)
        for b in F.bt.leaves():
            t, s = b.t, b.s
            rt = slice(t.start, t.start + t.size)
            rs = slice(s.start, s.start + s.size)
            if t is s:
                N = F.N[b.id]
                M = np.tril(N, -1) + np.eye(t.size) if base == "L" else np.triu(N)
                Y[rt] += M.T @ V[rt]
                continue
            lower = t.start > s.start
            if (base == "L") == lower:
                if b.kind == DENSE:
                    Y[rs] += F.N[b.id].T @ V[rt]
                else:
                    Y[rs] += F.B[b.id] @ (F.A[b.id].T @ V[rt])
        return Y
    Y = np.zeros_like(V)
    for b in F.bt.leaves():
        t, s = b.t, b.s
        rt = slice(t.start, t.start + t.size)
        rs = slice(s.start, s.start + s.size)
        if t is s:
            N = F.N[b.id]
            if part == "L":
                M = np.tril(N, -1) + np.eye(t.size)
            elif part == "R":
                M = np.triu(N)
            elif part == "Lc":
                M = np.tril(N)
            else:
                M = np.tril(N).T
            Y[rt] += M @ V[rt]
            continue
        lower = t.start > s.start
        if part in ("L", "Lc") and lower or part == "R" and not lower:
            if b.kind == DENSE:
                Y[rt] += F.N[b.id] @ V[rs]
            else:
                Y[rt] += F.A[b.id] @ (F.B[b.id].T @ V[rs])
        elif part == "LcT" and lower:
            # (L^T)_{s,t} = L_{t,s}^T  ->  Y[s] += L_{t,s}^T V[t]
            if b.kind == DENSE:
                Y[rs] += F.N[b.id].T @ V[rt]
            else:
                Y[rs] += F.B[b.id] @ (F.A[b.id].T @ V[rt])
    return Y


def probe_residual(G0: HMatrix, F: HMatrix, probes, kind="lr", shift=0.0):
    """||G v - L(R v)|| / ||G v|| (LR) or ||G v - L(L^T v)|| / ||G v|| (Cholesky),
    columns of `probes` in tree order; G0 = pre-factorization H-matrix."""
    from .hmatrix import matvec
    Gv = np.zeros_like(probes)
    matvec(G0, 1.0, probes, Gv)
    if shift:
        Gv = Gv + shift * probes
    if kind == "lr":
        LRv = apply_factor(F, "L", apply_factor(F, "R", probes))
    else:
        LRv = apply_factor(F, "Lc", apply_factor(F, "LcT", probes))
    return float(np.linalg.norm(Gv - LRv) / np.linalg.norm(Gv))


# ------------------------------------------------------------ solving with the factors

def solve_factor(F: HMatrix, part, V):
    """V <- op(F)^{-1} V (in place) by block substitution through the cluster
    tree: the inverse of apply_factor's operators, part in
      'L'   unit lower L (H-LR)        'R'   upper R (H-LR)
      'LT'  L^T (unit upper)           'RT'  R^T (lower)
      'Lc'  Cholesky factor L (lower)  'LcT' L^T (upper)
    Forward substitution for the lower operators (solve the t1 rows, subtract
    the (t2,t1) block's contribution with addeval / addevaltrans, solve t2),
    backward for the upper ones; dense diagonal leaves with
    scipy.linalg.solve_triangular.  Used for (L R)^{-1} in the preconditioner
    error of PAPER.md P:L1628-1629 (power iteration).
    Pinned by tests/test_oracle_factor.py against numpy.linalg.solve of the
    dense operator apply_factor(F, part, I)."""
    lower = part in ("L", "RT", "Lc")
    unit = part in ("L", "LT")
    G = F

    def rec(t, W):
        if t.leaf:
            N = G.N[_diag(G, t).id]
            if part in ("L", "Lc"):
                W[:] = sla.solve_triangular(N, W, lower=True, unit_diagonal=unit)
            elif part == "R":
                W[:] = sla.solve_triangular(N, W, lower=False)
            elif part == "RT":
                W[:] = sla.solve_triangular(N, W, lower=False, trans="T")
            else:   # LT, LcT: (lower N)^T
                W[:] = sla.solve_triangular(N, W, lower=True, trans="T", unit_diagonal=unit)
            return
        t1, t2 = t.sons
        W1, W2 = W[_rows(t, t1)], W[_rows(t, t2)]
        if lower:
            rec(t1, W1)
            if part == "RT":                       # (R^T)_(t2,t1) = R_(t1,t2)^T
                addevaltrans(G, G.bt.find(t1, t2), -1.0, W1, W2)
            else:                                  # L_(t2,t1)
                addeval(G, G.bt.find(t2, t1), -1.0, W1, W2)
            rec(t2, W2)
        else:
            rec(t2, W2)
            if part == "R":                        # R_(t1,t2)
                addeval(G, G.bt.find(t1, t2), -1.0, W2, W1)
            else:                                  # (L^T)_(t1,t2) = L_(t2,t1)^T
                addevaltrans(G, G.bt.find(t2, t1), -1.0, W2, W1)
            rec(t1, W1)

    rec(G.bt.root.t, V)
    return V


def precond_error(G0: HMatrix, F: HMatrix, kind="lr", iters=30, seed=0, v0=None):
    """Spectral norm estimate of E = I - (F)^{-1} G0 (the paper's
    "preconditioner error" ||I - G~^{-1} G||_2) by power
    iteration on E^T E: v <- E^T E v / ||.||, estimate ||E v|| (||v|| = 1).
    F = the in-place H-LR (kind 'lr': F = L R) or H-Cholesky (kind 'chol':
    F = L L^T of the symmetric G0).  E^T = I - G0^T F^{-T}.
    Pinned by tests/test_oracle_factor.py against numpy.linalg.norm(E, 2)."""
    from .hmatrix import matvec
    n = G0.n
    v = np.random.default_rng([1703, 9085, 5, seed]).standard_normal(n) if v0 is None else np.array(v0, float)
    v = v / np.linalg.norm(v)
    est = 0.0
    for _ in range(iters):
        gv = np.zeros(n)
        matvec(G0, 1.0, v, gv)
        if kind == "lr":
            solve_factor(F, "R", solve_factor(F, "L", gv))
        else:
            solve_factor(F, "LcT", solve_factor(F, "Lc", gv))
        w = v - gv
        est = float(np.linalg.norm(w))
        y = w.copy()
        if kind == "lr":                           # F^{-T} = L^{-T} R^{-T}
            solve_factor(F, "LT", solve_factor(F, "RT", y))
        else:
            solve_factor(F, "LcT", solve_factor(F, "Lc", y))
        z = np.zeros(n)
        matvec(G0, 1.0, y, z, trans=True)
        u = w - z
        nu = np.linalg.norm(u)
        if nu == 0.0:
            return 0.0
        v = u / nu
    return est
