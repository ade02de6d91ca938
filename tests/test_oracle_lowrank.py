"""Pins for TRUNC_eps / rkadd / rowmerge / rkmerge (§3).

Closed form (Eckart-Young): stacks built from A B^T = U diag(s) V^T
with PRESCRIBED singular values s, split into random exact terms (including
duplicated / cancelling columns, i.e. rank-deficient stacks).  The expected
rank k and error sqrt(sum_{i>k} s_i^2) are computed from s directly.
"""
import numpy as np
import pytest
from scipy.linalg import block_diag

from oracle.lowrank import TruncCtx, choose_rank, rkadd, rkmerge, rowmerge, trunc


def _orth(rng, m, k):
    q, _ = np.linalg.qr(rng.standard_normal((m, k)))
    return q


def prescribed_stack(rng, m, n, s, nterms, junk=0):
    """A, B (l columns) with A B^T = U diag(s) V^T exactly up to rounding.
    junk adds cancelling pairs [X, -X][Y, Y] (rank-deficient stack)."""
    q = len(s)
    U = _orth(rng, m, q)
    V = _orth(rng, n, q)
    # split columns of U diag(s) V^T into nterms groups, each mixed by an
    # invertible transform T: (U S T)(V T^-T)^T = U S V^T
    cuts = np.sort(rng.choice(np.arange(1, q), size=min(nterms - 1, q - 1), replace=False)) if q > 1 else []
    groups = np.split(np.arange(q), cuts)
    As, Bs = [], []
    for g in groups:
        T = rng.standard_normal((len(g), len(g))) + 3 * np.eye(len(g))
        As.append((U[:, g] * s[g]) @ T)
        Bs.append(V[:, g] @ np.linalg.inv(T).T)
    for _ in range(junk):
        X = rng.standard_normal((m, 2))
        Y = rng.standard_normal((n, 2))
        As += [X, -X]
        Bs += [Y, Y]
    return np.hstack(As), np.hstack(Bs)


def expected_rank(s, eps):
    tot = np.sum(s ** 2)
    for k in range(len(s) + 1):
        if np.sum(s[k:] ** 2) <= eps ** 2 * tot:
            return k
    return len(s)


@pytest.mark.parametrize("m,n,q,nterms,junk", [
    (60, 50, 12, 3, 0),      # thin route (l < min(m,n))
    (200, 80, 20, 8, 2),     # thin route, rank-deficient stack
    (30, 40, 25, 5, 3),      # dense route (l >= min(m,n))
    (16, 100, 16, 1, 4),     # wide, dense route
])
@pytest.mark.parametrize("eps", [1e-2, 1e-4, 1e-6])
def test_trunc_prescribed_sigma(m, n, q, nterms, junk, eps):
    rng = np.random.default_rng([m, n, q, int(-np.log10(eps))])
    s = 10.0 ** (-np.arange(q) / 3.0)
    A, B = prescribed_stack(rng, m, n, s, nterms, junk)
    ctx = TruncCtx(eps)
    Ak, Bk = trunc(A, B, ctx)
    k = expected_rank(s, eps)
    assert Ak.shape[1] == k and Bk.shape[1] == k
    M = A @ B.T
    err = np.linalg.norm(M - Ak @ Bk.T)
    np.testing.assert_allclose(err, np.sqrt(np.sum(s[k:] ** 2)), rtol=1e-9, atol=1e-13)
    # left factor orthonormal (Fig. 2: C <- U(:,1:k))
    np.testing.assert_allclose(Ak.T @ Ak, np.eye(k), atol=1e-13)


def test_trunc_clustered_sigma():
    rng = np.random.default_rng(7)
    s = np.array([1.0, 1.0, 1.0, 0.5, 0.5, 1e-3, 1e-3, 1e-9])
    A, B = prescribed_stack(rng, 40, 30, s, 3, 1)
    Ak, Bk = trunc(A, B, TruncCtx(1e-2))
    k = expected_rank(s, 1e-2)
    assert k == 5 and Ak.shape[1] == 5
    np.testing.assert_allclose(np.linalg.norm(A @ B.T - Ak @ Bk.T), np.sqrt(2e-6 + 1e-18), rtol=1e-8)


def test_choose_rank_special_cases():
    assert choose_rank(np.zeros(4), 1e-4)[0] == 0
    assert choose_rank(np.array([]), 1e-4)[0] == 0
    assert choose_rank(np.array([3.0, 2.0, 1.0, 0.0]), 0.0)[0] == 3
    # sum_{i>k} s^2 <= eps^2 sum s^2 : s=(1, .1), total 1.01; eps=.1 -> tail(1)=.01 <= .0101
    assert choose_rank(np.array([1.0, 0.1]), 0.1)[0] == 1
    assert choose_rank(np.array([1.0, 0.1]), 0.0995)[0] == 2


def test_trunc_eps0_exact_and_empty():
    rng = np.random.default_rng(1)
    A = rng.standard_normal((20, 5))
    B = rng.standard_normal((15, 5))
    Ak, Bk = trunc(A, B, TruncCtx(0.0))
    assert Ak.shape[1] == 5
    np.testing.assert_allclose(Ak @ Bk.T, A @ B.T, atol=1e-13)
    Ak, Bk = trunc(np.zeros((7, 0)), np.zeros((9, 0)), TruncCtx(1e-4))
    assert Ak.shape == (7, 0) and Bk.shape == (9, 0)


def test_rkadd_cancellation_and_alpha0():
    rng = np.random.default_rng(2)
    R = (rng.standard_normal((30, 4)), rng.standard_normal((25, 4)))
    A, B = rkadd(-1.0, R, R, TruncCtx(1e-12))
    assert A.shape[1] == 0 or np.linalg.norm(A @ B.T) <= 1e-12 * np.linalg.norm(R[0] @ R[1].T)
    R2 = (rng.standard_normal((30, 3)), rng.standard_normal((25, 3)))
    A, B = rkadd(0.0, R, R2, TruncCtx(0.0))
    np.testing.assert_allclose(A @ B.T, R2[0] @ R2[1].T, atol=1e-12)


def test_rkadd_matches_dense_truncation():
    """SPEC rkadd equivalence: equals the optimal truncation of the dense sum."""
    rng = np.random.default_rng(3)
    R1 = (rng.standard_normal((40, 2)), rng.standard_normal((35, 2)))
    R2 = (rng.standard_normal((40, 2)), rng.standard_normal((35, 2)))
    S = R2[0] @ R2[1].T + 0.7 * R1[0] @ R1[1].T
    sv = np.linalg.svd(S, compute_uv=False)
    eps = 1.5 * sv[3] / np.linalg.norm(sv)  # forces a cut inside the rank-4 sum
    A, B = rkadd(0.7, R1, R2, TruncCtx(eps))
    k = expected_rank(sv[:4], eps)
    assert A.shape[1] == k
    assert k < 4
    np.testing.assert_allclose(np.linalg.norm(S - A @ B.T), np.sqrt(np.sum(sv[k:] ** 2)), rtol=1e-9)


def test_rowmerge_rkmerge_dense_assembly():
    rng = np.random.default_rng(4)
    # 2x3 grid of random rank-2 blocks
    rows, cols = [13, 17], [9, 11, 8]
    grid = [[(rng.standard_normal((m, 2)), rng.standard_normal((n, 2))) for n in cols] for m in rows]
    D = np.block([[a @ b.T for a, b in row] for row in grid])
    A, B = rkmerge(grid, TruncCtx(0.0))
    np.testing.assert_allclose(A @ B.T, D, atol=1e-12 * np.linalg.norm(D))
    # truncating merge: error equals Eckart-Young of the dense block matrix
    sv = np.linalg.svd(D, compute_uv=False)
    eps = 0.5
    A, B = rowmerge([(np.hstack([g[0] for g in grid[0]]), block_diag(*[g[1] for g in grid[0]]))], TruncCtx(eps))
    # single part = TRUNC of itself
    D0 = np.hstack([a @ b.T for a, b in grid[0]])
    s0 = np.linalg.svd(D0, compute_uv=False)
    k = expected_rank(s0, eps)
    assert A.shape[1] == k < 6
    np.testing.assert_allclose(np.linalg.norm(D0 - A @ B.T), np.sqrt(np.sum(s0[k:] ** 2)), rtol=1e-9)
    # global rank-1 2x2 grid -> rank-1 result reproducing it
    u = rng.standard_normal(30)
    v = rng.standard_normal(20)
    g1 = [[(u[:12, None], v[:7, None]), (u[:12, None], v[7:, None])],
          [(u[12:, None], v[:7, None]), (u[12:, None], v[7:, None])]]
    A, B = rkmerge(g1, TruncCtx(1e-10))
    assert A.shape[1] == 1
    np.testing.assert_allclose(A @ B.T, np.outer(u, v), atol=1e-12 * np.linalg.norm(u) * np.linalg.norm(v))


def test_many_random_truncations():
    """>= 100 randomized instances (SPEC acceptance 2)."""
    rng = np.random.default_rng(5)
    for it in range(120):
        m, n = rng.integers(2, 40, size=2)
        q = int(rng.integers(1, min(m, n) + 1))
        s = np.sort(rng.uniform(0, 1, q) ** 4)[::-1]
        A, B = prescribed_stack(rng, m, n, s, int(rng.integers(1, 5)), int(rng.integers(0, 2)))
        eps = float(10.0 ** rng.uniform(-8, -1))
        Ak, Bk = trunc(A, B, TruncCtx(eps))
        k = expected_rank(s, eps)
        # skip razor-thin decisions (tail within 1e-8 relative of threshold)
        thr = eps ** 2 * np.sum(s ** 2)
        tails = [np.sum(s[j:] ** 2) for j in range(q + 1)]
        if any(abs(tails[j] - thr) <= 1e-8 * thr for j in range(q + 1)):
            continue
        assert Ak.shape[1] == k, it
        np.testing.assert_allclose(np.linalg.norm(A @ B.T - Ak @ Bk.T), np.sqrt(tails[k]),
                                   rtol=1e-7, atol=1e-14 * np.linalg.norm(A) * np.linalg.norm(B))
