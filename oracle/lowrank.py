"""Low-rank truncation algebra (§3).

TRUNC_eps(A, B): the eps-truncated SVD of the EXACT matrix A B^T.
  * Route: the paper's "Truncation" paragraph: thin QR of B,
    A_hat = A R_B^T, thin SVD of A_hat, V = Q_B V_hat.  Used when
    l < min(m, n); otherwise (l >= min(m,n), the stack is not thin) the SVD
    of the dense A B^T -- same matrix, same singular values.
  * "Choose new rank k" is the reading of SURVEY §8(c) #1:
    k = smallest k >= 0 with sum_{i>k} s_i^2 <= eps^2 sum_i s_i^2 (relative
    Frobenius, block-local, tails accumulated from the smallest s upward,
    compared in FP64; k = 0 if the total is 0).
  * Output convention of Fig. 2: left factor U_k (orthonormal),
    right factor V_k Sigma_k.

Pinned by tests/test_oracle_lowrank.py: prescribed-sigma stacks (closed-form
Eckart-Young error and rank), rkadd(-1,R,R) -> rank 0,
rowmerge/rkmerge against the dense assembly, exactness at eps = 0.
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla

U_ROUND = 2.0 ** -53


class TruncCtx:
    """Truncation control + instrumentation (SPEC-style counters)."""

    def __init__(self, eps, log_near=True, near_rel=1e-10, near_abs_ulps=64.0):
        self.eps = float(eps)
        self.count = 0          # number of TRUNC calls
        self.cols = 0           # sum of stacked widths l
        self.log_near = log_near
        self.near_rel = near_rel
        self.near_abs_ulps = near_abs_ulps
        self.near = []          # (count index, tag, k, s) of near-threshold decisions
        self.tag = None         # optional caller-provided label of the current truncation
        self.forced = {}        # count index -> forced rank (forced-rank replay)
        self.ranks = []         # per call: (tag, k)
        self.counter = None     # optional oracle.flops.ConventionCounter (timing reports only)

    def record(self, m, n, l, k):
        self.ranks.append((self.tag, k))
        if self.counter is not None:
            self.counter.on_trunc(m, n, l, k)


def choose_rank(s, eps):
    """Rank rule of SURVEY §8(c) O4 (reading #1 of "Choose new rank k")."""
    q = len(s)
    tail = np.zeros(q + 1)
    acc = 0.0
    for i in range(q - 1, -1, -1):
        acc = acc + s[i] * s[i]
        tail[i] = acc
    total = tail[0]
    if total == 0.0:
        return 0, tail
    thr = (eps * eps) * total
    for k in range(q + 1):
        if tail[k] <= thr:
            return k, tail
    return q, tail  # unreachable: tail[q] = 0


def _near(ctx, s, k, tail):
    if not ctx.log_near or len(s) == 0 or tail[0] == 0.0:
        return False
    thr = np.sqrt((ctx.eps * ctx.eps) * tail[0])
    band = max(ctx.near_rel * thr, ctx.near_abs_ulps * U_ROUND * s[0] * np.sqrt(len(s)))
    for j in (k - 1, k):
        if 0 <= j <= len(s) and abs(np.sqrt(tail[j]) - thr) <= band:
            return True
    return False


def _svd(M):
    return sla.svd(M, full_matrices=False, lapack_driver="gesvd")


def trunc(A, B, ctx: TruncCtx):
    """TRUNC_eps(A, B) -> (U_k, V_k Sigma_k) of the exact A B^T."""
    A = np.asarray(A, np.float64)
    B = np.asarray(B, np.float64)
    m, l = A.shape
    n = B.shape[0]
    assert B.shape[1] == l
    idx = ctx.count
    ctx.count += 1
    ctx.cols += l
    if l == 0 or m == 0 or n == 0:
        ctx.record(m, n, l, 0)
        return np.zeros((m, 0)), np.zeros((n, 0))
    if l < min(m, n):
        QB, RB = np.linalg.qr(B)              # thin QR  B = Q_B R_B
        Ahat = A @ RB.T                       # A_hat = A R_B^*
        U, s, Vh = _svd(Ahat)                 # A_hat = U Sigma V_hat^*
        k, tail = choose_rank(s, ctx.eps)
        k = ctx.forced.get(idx, k)
        if ctx.log_near and _near(ctx, s, k, tail):
            ctx.near.append((idx, ctx.tag, k, s.copy()))
        ctx.record(m, n, l, k)
        return U[:, :k].copy(), QB @ (Vh[:k].T * s[:k])   # V = Q_B V_hat
    S = A @ B.T
    U, s, Vh = _svd(S)
    k, tail = choose_rank(s, ctx.eps)
    k = ctx.forced.get(idx, k)
    if ctx.log_near and _near(ctx, s, k, tail):
        ctx.near.append((idx, ctx.tag, k, s.copy()))
    ctx.record(m, n, l, k)
    return U[:, :k].copy(), Vh[:k].T * s[:k]


def rkadd(alpha, R1, R2, ctx):
    """Fig. 2: R2 <- trunc(R2 + alpha R1) via the stack
    [alpha A, C] [B, D]^T (QR of [B D], SVD of [alpha A, C] R_B^*)."""
    A, B = R1
    C, D = R2
    return trunc(np.hstack([alpha * A, C]), np.hstack([B, D]), ctx)


def rowmerge(parts, ctx):
    """Fig. 4 rowmerge: truncation of the exact horizontal
    concatenation [R_1 ... R_p] (R_j = A_j B_j^T share the row set).
    Literal: QR of every B_j, SVD of [A_1 R_{B,1}^* ... A_p R_{B,p}^*],
    B = blockdiag(Q_{B,j}) V_hat Sigma~."""
    m = parts[0][0].shape[0]
    ns = [p[1].shape[0] for p in parts]
    Qs, Ahats = [], []
    for A, B in parts:
        assert A.shape[0] == m
        Q, R = np.linalg.qr(B)
        Qs.append(Q)
        Ahats.append(A @ R.T)
    Ahat = np.hstack(Ahats)
    idx = ctx.count
    ctx.count += 1
    lsum = sum(p[0].shape[1] for p in parts)
    ctx.cols += lsum
    if Ahat.shape[1] == 0 or m == 0:
        ctx.record(m, sum(ns), lsum, 0)
        return np.zeros((m, 0)), np.zeros((sum(ns), 0))
    U, s, Vh = _svd(Ahat)
    k, tail = choose_rank(s, ctx.eps)
    k = ctx.forced.get(idx, k)
    if ctx.log_near and _near(ctx, s, k, tail):
        ctx.near.append((idx, ctx.tag, k, s.copy()))
    ctx.record(m, sum(ns), lsum, k)
    W = Vh[:k].T * s[:k]
    Bout = np.zeros((sum(ns), k))
    r0 = c0 = 0
    for Q in Qs:
        Bout[r0:r0 + Q.shape[0]] = Q @ W[c0:c0 + Q.shape[1]]
        r0 += Q.shape[0]
        c0 += Q.shape[1]
    return U[:, :k].copy(), Bout


def rkmerge(grid, ctx):
    """Fig. 4 rkmerge: per block column j, rowmerge of the
    adjoints R_{1j}^*, ..., R_{pj}^* (the exact vertical stack), then
    rowmerge of the block columns (the exact horizontal row).
    grid[i][j] = (A_ij, B_ij)."""
    p = len(grid)
    q = len(grid[0])
    cols = []
    for j in range(q):
        # adjoint R_ij^* = B_ij A_ij^*  ->  rowmerge over i
        Bt, At = rowmerge([(grid[i][j][1], grid[i][j][0]) for i in range(p)], ctx)
        cols.append((At, Bt))   # R_j = At Bt^T  (#t x #r_j)
    return rowmerge(cols, ctx)


def dense_of(R):
    A, B = R
    return A @ B.T
