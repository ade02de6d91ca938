"""H-matrix multiplication Z <- blocktrunc(Z + alpha X Y)  (§4-5).

Three schedules:
  S0  standard immediate-update product: every elementary
      product is added with rkupdate at once; temporaries + rkmerge below
      admissible Z leaves.
  S1  literal accumulated product, Figs. 5-7 verbatim: every evaluated
      term is rkadd-ed into R_hat at once.
  S2  level-batched accumulated product -- the GPU parity schedule
      (reading #9 of SURVEY §8(c)): evaluated terms are kept EXACT in the
      accumulator and truncated once, either when the accumulator is split
      (reduce = T1) or when it is flushed into a leaf (T2 real admissible
      leaf, T3 virtual leaf), plus the rkmerge truncations (T4).

Common readings: alpha applied once per product, folded into A_hat (#2,
P:L986 vs L991); Fig. 7 P:L1079 flushes into Z|_{t' x r'} (#5); the
"#t <= #s" tie takes the identity branch (#11); son loops row-major over
sons(t) x sons(r), then pending order, then s' (#12).

Pinned by tests/test_oracle_product.py: eps = 0 product equals the dense
Z + alpha X Y to 1e-12 on tiny n (all Fig. 5 and Fig. 7 branches hit);
content conservation; addproduct calls == product-tree nodes;
each Z leaf updated exactly once in S2; S0/S1/S2 agree within
the eps bound; relative error vs dense at eps = 1e-4.
"""
from __future__ import annotations

import numpy as np

from .hmatrix import HMatrix, addeval, addevaltrans, rkupdate
from .lowrank import TruncCtx, rkadd, rkmerge, trunc
from .trees import ADM, DENSE, SUB


class Stats:
    def __init__(self):
        self.addproduct = 0        # calls of addproduct (Fig. 5)
        self.evaluated = 0         # products evaluated into low-rank terms
        self.pending = 0           # products deferred
        self.branch = [0, 0, 0, 0, 0, 0, 0, 0]  # Fig 5 branches (see evaluate)
        self.leaf_updates = {}     # Z leaf id -> number of T2 / dense adds
        self.flush_branch = {}     # Fig 7 branch name -> count
        self.virtual_nodes = 0
        self.merges = 0

    def fb(self, name):
        self.flush_branch[name] = self.flush_branch.get(name, 0) + 1


# --------------------------------------------------------------- Fig. 5

def evaluate(alpha, bx, by, X: HMatrix, Y: HMatrix, st: Stats | None = None, counter=None):
    """Low-rank factorization A_hat B_hat^* = alpha X|_{ts} Y|_{sr} of a product
    whose (t,s) or (s,r) block is a leaf, in Fig. 5's printed branch order
    (P:L969-1006).  Returns (A_hat, B_hat) or None if the product is pending.
    """
    t, s = bx.t, bx.s
    r = by.s
    if bx.kind == DENSE:                                   # (t,s) in L^-
        N = X.N[bx.id]
        if t.size <= s.size:                               # A_hat = I_t
            Ah = alpha * np.eye(t.size)
            Bh = np.zeros((r.size, t.size))
            addevaltrans(Y, by, 1.0, N.T, Bh)              # B_hat += Y^* N_X^*
            br = 0
        else:                                              # A_hat = N_X
            Ah = alpha * N
            Bh = np.zeros((r.size, s.size))
            addevaltrans(Y, by, 1.0, np.eye(s.size), Bh)   # B_hat += Y^* I
            br = 1
    elif by.kind == DENSE:                                 # (s,r) in L^-
        N = Y.N[by.id]
        if r.size <= s.size:                               # B_hat = I_r
            Bh = np.eye(r.size)
            Ah = np.zeros((t.size, r.size))
            addeval(X, bx, alpha, N, Ah)                   # A_hat += alpha X N_Y
            br = 2
        else:                                              # B_hat = N_Y^*
            Bh = N.T.copy()
            Ah = np.zeros((t.size, s.size))
            addeval(X, bx, alpha, np.eye(s.size), Ah)      # A_hat += alpha X I
            br = 3
    elif bx.kind == ADM:                                   # (t,s) in L^+
        Ah = alpha * X.A[bx.id]
        Bh = np.zeros((r.size, Ah.shape[1]))
        addevaltrans(Y, by, 1.0, X.B[bx.id], Bh)           # B_hat += Y^* B_X
        br = 4
    elif by.kind == ADM:                                   # (s,r) in L^+
        Bh = Y.B[by.id].copy()
        Ah = np.zeros((t.size, Bh.shape[1]))
        addeval(X, bx, alpha, Y.A[by.id], Ah)              # A_hat += alpha X A_Y
        br = 5
    else:
        if st is not None:
            st.pending += 1
        return None
    if st is not None:
        st.evaluated += 1
        st.branch[br] += 1
    if counter is not None:   # convention flops of the addeval/addevaltrans just done
        H, blk = (Y, by) if br in (0, 1, 4) else (X, bx)
        counter.on_eval(H, blk, Ah.shape[1], br in (1, 3))
    return Ah, Bh


# ------------------------------------------------------ Z targets

class ZReal:
    """A node of Z's block tree."""
    virtual = False

    def __init__(self, h: HMatrix, b):
        self.h, self.b = h, b
        self.t, self.r = b.t, b.s

    @property
    def kind(self):
        return self.b.kind

    def son(self, i, j):
        return ZReal(self.h, self.b.son(i, j))

    def factors(self):
        return self.h.A[self.b.id], self.h.B[self.b.id]

    def set_factors(self, A, B):
        self.h.A[self.b.id], self.h.B[self.b.id] = A, B

    def key(self):
        return ("real", self.b.id)


class ZVirt:
    """Temporary low-rank matrix Z~_{t',r'} below an admissible leaf (Fig. 7,
    P:L1082-1084): a copy of the restriction of the parent's factors."""
    virtual = True
    kind = ADM

    def __init__(self, t, r, A, B):
        self.t, self.r = t, r
        self.A, self.B = A, B

    def factors(self):
        return self.A, self.B

    def set_factors(self, A, B):
        self.A, self.B = A, B

    def key(self):
        return ("virt", self.t.id, self.r.id)


def _virtual_sons(z):
    A, B = z.factors()
    t, r = z.t, z.r
    grid = []
    for ti in t.sons:
        row = []
        for rj in r.sons:
            a = A[ti.start - t.start:ti.start - t.start + ti.size].copy()
            bb = B[rj.start - r.start:rj.start - r.start + rj.size].copy()
            row.append(ZVirt(ti, rj, a, bb))
        grid.append(row)
    return grid


# ------------------------------------------------------ S2 accumulator

class Acc2:
    """Accumulator (R_hat_{t,r}, P_{t,r}) of §4, S2 form:
    base (A0,B0) already truncated, exact terms [(A_hat_i, B_hat_i)], pending
    [(alpha, bx, by)]."""

    def __init__(self, t, r, base=None):
        self.t, self.r = t, r
        self.base = base
        self.terms = []
        self.pending = []

    def stack(self):
        As, Bs = [], []
        if self.base is not None:
            As.append(self.base[0])
            Bs.append(self.base[1])
        for a, b in self.terms:
            As.append(a)
            Bs.append(b)
        if not As:
            return np.zeros((self.t.size, 0)), np.zeros((self.r.size, 0))
        return np.hstack(As), np.hstack(Bs)

    def content_lowrank(self):
        """dense(base) + sum of terms (exact; no subtraction)."""
        A, B = self.stack()
        return A @ B.T


class S2:
    """Level-batched accumulated product (the GPU parity schedule)."""

    def __init__(self, X, Y, ctx: TruncCtx, stats: Stats | None = None, counter=None):
        self.X, self.Y, self.ctx = X, Y, ctx
        self.st = stats or Stats()
        self.counter = counter
        if counter is not None:
            ctx.counter = counter

    def addproduct(self, acc: Acc2, alpha, bx, by, X=None, Y=None):
        """Fig. 5, S2: evaluated terms are appended exactly.
        X, Y: the H-matrices the blocks bx, by belong to (default: the
        product's X and Y; the inversion of Fig. 8 mixes G and the auxiliary
        H); a pending product remembers them."""
        X = self.X if X is None else X
        Y = self.Y if Y is None else Y
        self.st.addproduct += 1
        ev = evaluate(alpha, bx, by, X, Y, self.st, self.counter)
        if ev is None:
            acc.pending.append((alpha, bx, by, X, Y))
        else:
            acc.terms.append(ev)

    def reduce(self, acc: Acc2, tag):
        """T1: base <- TRUNC([A0, A_hat_i], [B0, B_hat_i]) if terms exist."""
        if acc.terms:
            A, B = acc.stack()
            self.ctx.tag = ("T1",) + tag
            acc.base = trunc(A, B, self.ctx)
            acc.terms = []

    def split(self, acc: Acc2, tag, lower_only=False):
        """Fig. 6 after reduce: sons inherit restrictions of the
        base, pending products are expanded over sons(s).
        lower_only (H-Cholesky): strictly upper sons are not created."""
        self.reduce(acc, tag)
        t, r = acc.t, acc.r
        grid = []
        for i, ti in enumerate(t.sons):
            row = []
            for j, rj in enumerate(r.sons):
                if lower_only and ti.start < rj.start:
                    row.append(None)
                    continue
                base = None
                if acc.base is not None:
                    A0, B0 = acc.base
                    base = (A0[ti.start - t.start:ti.start - t.start + ti.size],
                            B0[rj.start - r.start:rj.start - r.start + rj.size])
                son = Acc2(ti, rj, base)
                for alpha, bx, by, X, Y in acc.pending:
                    for l in range(len(bx.s.sons)):
                        self.addproduct(son, alpha, bx.son(i, l), by.son(l, j), X, Y)
                row.append(son)
            grid.append(row)
        return grid

    def flush(self, acc: Acc2, z):
        """Fig. 7 in S2 form (SURVEY O6 branches i-v)."""
        tag = (z.t.id, z.r.id)
        if not acc.pending:
            if z.virtual or z.kind == ADM:                      # (i) T2 / T3
                self.st.fb("i_virtual" if z.virtual else "i_adm")
                AZ, BZ = z.factors()
                A, B = acc.stack()
                self.ctx.tag = ("T3" if z.virtual else "T2",) + tag
                z.set_factors(*trunc(np.hstack([AZ, A]), np.hstack([BZ, B]), self.ctx))
                if not z.virtual:
                    self._leaf_update(z.b.id)
            elif z.kind == DENSE:                               # (ii) exact add
                self.st.fb("ii_dense")
                A, B = acc.stack()
                z.h.N[z.b.id] += A @ B.T
                if self.counter is not None:
                    self.counter.on_dense(A.shape[0], B.shape[0], A.shape[1])
                self._leaf_update(z.b.id)
            else:                                               # (iii)
                self.st.fb("iii_sub")
                self.reduce(acc, tag)
                if acc.base is not None:
                    self._rkupdate_s2(z.h, z.b, acc.base[0], acc.base[1])
                else:
                    self._rkupdate_s2(z.h, z.b, np.zeros((z.t.size, 0)), np.zeros((z.r.size, 0)))
            acc.base, acc.terms, acc.pending = None, [], []
            return
        if not z.virtual and z.kind == SUB:                      # (iv)
            self.st.fb("iv_sub")
            grid = self.split(acc, tag)
            for i in range(len(grid)):
                for j in range(len(grid[i])):
                    self.flush(grid[i][j], z.son(i, j))
        elif z.virtual or z.kind == ADM:                         # (v)
            self.st.fb("v_virtual" if z.virtual else "v_adm")
            zs = _virtual_sons(z)
            self.st.virtual_nodes += sum(len(row) for row in zs)
            grid = self.split(acc, tag)
            for i in range(len(grid)):
                for j in range(len(grid[i])):
                    self.flush(grid[i][j], zs[i][j])
            self.ctx.tag = ("T4",) + tag
            self.st.merges += 1
            z.set_factors(*rkmerge([[v.factors() for v in row] for row in zs], self.ctx))
            if not z.virtual:
                self._leaf_update(z.b.id)
        else:
            raise AssertionError("flush: pending products into a dense leaf (impossible, SURVEY O6 vi)")
        acc.base, acc.terms, acc.pending = None, [], []

    def _leaf_update(self, bid):
        self.st.leaf_updates[bid] = self.st.leaf_updates.get(bid, 0) + 1

    def _rkupdate_s2(self, h, b, A, B):
        """Branch (iii): each Z leaf of the subtree gets T2 with the restricted
        base, or an exact dense add (Fig. 3 recursion)."""
        if b.kind == DENSE:
            h.N[b.id] += A @ B.T
            self._leaf_update(b.id)
        elif b.kind == ADM:
            self.ctx.tag = ("T2", b.t.id, b.s.id)
            h.A[b.id], h.B[b.id] = trunc(np.hstack([h.A[b.id], A]), np.hstack([h.B[b.id], B]), self.ctx)
            self._leaf_update(b.id)
        else:
            t0, s0 = b.t.start, b.s.start
            for c in b.sons:
                self._rkupdate_s2(h, c, A[c.t.start - t0:c.t.start - t0 + c.t.size],
                                  B[c.s.start - s0:c.s.start - s0 + c.s.size])


def addmul_s2(alpha, X: HMatrix, Y: HMatrix, Z: HMatrix, eps, ctx=None, stats=None, counter=None):
    """Z <- blocktrunc(Z + alpha X Y) with accumulated updates: addproduct for
    the root of the product tree, then flush (Theorem)."""
    ctx = ctx or TruncCtx(eps)
    alg = S2(X, Y, ctx, stats, counter)
    bt = Z.bt
    root = bt.root
    acc = Acc2(root.t, root.s)
    alg.addproduct(acc, alpha, X.bt.root, Y.bt.root)
    alg.flush(acc, ZReal(Z, root))
    return Z, ctx, alg.st


# ------------------------------------------------------ S1 literal

class Acc1:
    def __init__(self, t, r, R=None):
        self.t, self.r = t, r
        self.R = R if R is not None else (np.zeros((t.size, 0)), np.zeros((r.size, 0)))
        self.pending = []


class S1:
    """Figs. 5-7 verbatim: evaluated terms rkadd-ed into R_hat at once."""

    def __init__(self, X, Y, ctx, stats=None):
        self.X, self.Y, self.ctx = X, Y, ctx
        self.st = stats or Stats()

    def addproduct(self, acc, alpha, bx, by):
        self.st.addproduct += 1
        ev = evaluate(alpha, bx, by, self.X, self.Y, self.st)
        if ev is None:
            acc.pending.append((alpha, bx, by))
        else:
            self.ctx.tag = ("rkadd", acc.t.id, acc.r.id)
            acc.R = rkadd(1.0, ev, acc.R, self.ctx)   # alpha already in A_hat

    def split(self, acc):
        t, r = acc.t, acc.r
        A, B = acc.R
        grid = []
        for i, ti in enumerate(t.sons):
            row = []
            for j, rj in enumerate(r.sons):
                son = Acc1(ti, rj, (A[ti.start - t.start:ti.start - t.start + ti.size],
                                    B[rj.start - r.start:rj.start - r.start + rj.size]))
                for alpha, bx, by in acc.pending:
                    for l in range(len(bx.s.sons)):
                        self.addproduct(son, alpha, bx.son(i, l), by.son(l, j))
                row.append(son)
            grid.append(row)
        return grid

    def flush(self, acc, z):
        if not acc.pending:
            A, B = acc.R
            if z.virtual:
                AZ, BZ = z.factors()
                self.ctx.tag = ("rkadd", z.t.id, z.r.id)
                z.set_factors(*rkadd(1.0, (A, B), (AZ, BZ), self.ctx))
            else:
                rkupdate(z.h, z.b, 1.0, A, B, self.ctx)
            return
        if not z.virtual and z.kind == SUB:
            grid = self.split(acc)
            for i in range(len(grid)):
                for j in range(len(grid[i])):
                    self.flush(grid[i][j], z.son(i, j))
        elif z.virtual or z.kind == ADM:
            zs = _virtual_sons(z)
            grid = self.split(acc)
            for i in range(len(grid)):
                for j in range(len(grid[i])):
                    self.flush(grid[i][j], zs[i][j])
            self.ctx.tag = ("merge", z.t.id, z.r.id)
            z.set_factors(*rkmerge([[v.factors() for v in row] for row in zs], self.ctx))
        else:
            raise AssertionError("flush: pending products into a dense leaf")


def addmul_s1(alpha, X, Y, Z, eps, ctx=None, stats=None):
    ctx = ctx or TruncCtx(eps)
    alg = S1(X, Y, ctx, stats)
    root = Z.bt.root
    acc = Acc1(root.t, root.s)
    alg.addproduct(acc, alpha, X.bt.root, Y.bt.root)
    alg.flush(acc, ZReal(Z, root))
    return Z, ctx, alg.st


# ------------------------------------------------------ S0 standard

def addmul_s0(alpha, X, Y, Z, eps, ctx=None, stats=None):
    """Standard product: rkupdate immediately; temporaries and
    rkmerge where (t,r) is an admissible leaf."""
    ctx = ctx or TruncCtx(eps)
    st = stats or Stats()

    def update(z, A, B):
        if z.virtual:
            AZ, BZ = z.factors()
            ctx.tag = ("rkadd", z.t.id, z.r.id)
            z.set_factors(*rkadd(1.0, (A, B), (AZ, BZ), ctx))
        else:
            rkupdate(z.h, z.b, 1.0, A, B, ctx)

    def mul(bx, by, z):
        st.addproduct += 1
        ev = evaluate(alpha, bx, by, X, Y, st)
        if ev is not None:
            update(z, *ev)
            return
        t, s, r = bx.t, bx.s, by.s
        if not z.virtual and z.kind == SUB:
            for i in range(len(t.sons)):
                for j in range(len(r.sons)):
                    zz = z.son(i, j)
                    for l in range(len(s.sons)):
                        mul(bx.son(i, l), by.son(l, j), zz)
        elif z.virtual or z.kind == ADM:
            zs = _virtual_sons(z)
            for i in range(len(t.sons)):
                for j in range(len(r.sons)):
                    for l in range(len(s.sons)):
                        mul(bx.son(i, l), by.son(l, j), zs[i][j])
            ctx.tag = ("merge", z.t.id, z.r.id)
            z.set_factors(*rkmerge([[v.factors() for v in row] for row in zs], ctx))
        else:
            raise AssertionError("standard product: subdivided product into a dense leaf")

    mul(X.bt.root, Y.bt.root, ZReal(Z, Z.bt.root))
    return Z, ctx, st


# ------------------------------------------------------ product tree

def product_tree_nodes(btx, bty):
    """Enumerate T_{IxJxK} (Def. P:L1151-1178) as (t,s,r) id triples."""
    out = []
    stack = [(btx.root, bty.root)]
    while stack:
        bx, by = stack.pop()
        out.append((bx.t.id, bx.s.id, by.s.id))
        if bx.leaf or by.leaf:
            continue
        for i in range(len(bx.t.sons)):
            for j in range(len(by.s.sons)):
                for l in range(len(bx.s.sons)):
                    stack.append((bx.son(i, l), by.son(l, j)))
    return out
