"""Pins for the H-LR / H-Cholesky oracle (oracle/factor.py, readings O8/O9).

  * eps = 0 on tiny n: L R = G and L L^T = G (dense assembly of the factors,
    independent of the recursion) to 1e-12.
  * block-diagonal input (all off-diagonal blocks zero): the factors are the
    blockwise dense LU / Cholesky factors.
  * leaf LU equals scipy.linalg.lu when scipy's permutation is the identity.
  * eps = 1e-4: probe residual ||G v - L(R v)|| / ||G v|| <= 50 eps (SURVEY #21).
  * pivot breakdown raises PivotError naming the cluster.
"""
import numpy as np
import pytest
import scipy.linalg as sla

from hm_inputs import probe_vectors, sphere_points
from oracle import kernel as K
from oracle.factor import PivotError, apply_factor, chol, chol_with_restart, lr, lu_nopivot, probe_residual
from oracle.hmatrix import Problem, build


def _prob(L, leaf, kernel=K.KERNEL_SLP):
    x, w = sphere_points(L)
    return Problem(x, w, leaf, 2.0, kernel=kernel)


@pytest.mark.parametrize("L,leaf", [(1, 4), (2, 8)])
def test_lr_exact_eps0(L, leaf):
    P = _prob(L, leaf)
    G = build(P, 0.0)
    Gd = G.to_dense()
    F, fo = lr(G.clone(), 0.0)
    n = P.ct.n
    I = np.eye(n)
    Ld = apply_factor(F, "L", I)
    Rd = apply_factor(F, "R", I)
    assert np.allclose(np.triu(Ld, 1), 0) and np.allclose(np.diag(Ld), 1)
    assert np.allclose(np.tril(Rd, -1), 0)
    assert np.linalg.norm(Ld @ Rd - Gd) <= 1e-12 * np.linalg.norm(Gd)
    # equals the dense (unpivoted) LU of the same matrix
    Lr, Rr = _dense_lu(Gd)
    assert np.linalg.norm(Ld - Lr) <= 1e-10 * np.linalg.norm(Lr)


def _dense_lu(A):
    N = A.copy()
    lu_nopivot(N)
    return np.tril(N, -1) + np.eye(len(N)), np.triu(N)


@pytest.mark.parametrize("L,leaf", [(1, 4), (2, 8)])
def test_chol_exact_eps0(L, leaf):
    P = _prob(L, leaf, K.KERNEL_SLP_SYM)
    G = build(P, 0.0)
    Gd = G.to_dense()
    F, fo = chol(G.clone(), 0.0)
    Ld = apply_factor(F, "Lc", np.eye(P.ct.n))
    assert np.allclose(np.triu(Ld, 1), 0)
    assert np.linalg.norm(Ld @ Ld.T - Gd) <= 1e-12 * np.linalg.norm(Gd)
    np.testing.assert_allclose(Ld, np.linalg.cholesky(Gd), atol=1e-11 * np.abs(Ld).max())


def test_block_diagonal_input():
    P = _prob(2, 8)
    G = build(P, 0.0)
    for k in G.A:
        G.A[k] = G.A[k][:, :0]
        G.B[k] = G.B[k][:, :0]
    for b in P.bt.leaves():
        if b.kind == 2 and b.t is not b.s:
            G.N[b.id][:] = 0.0
    Gd = G.to_dense()
    F, _ = lr(G.clone(), 1e-4)
    Ld = apply_factor(F, "L", np.eye(P.ct.n))
    Rd = apply_factor(F, "R", np.eye(P.ct.n))
    Lr, Rr = _dense_lu(Gd)
    np.testing.assert_allclose(Ld, Lr, atol=1e-12)
    np.testing.assert_allclose(Rd, Rr, atol=1e-12 * np.abs(Rr).max())


def test_leaf_lu_matches_scipy():
    rng = np.random.default_rng(1)
    A = rng.standard_normal((20, 20)) + 40 * np.eye(20)   # diagonally dominant: scipy pivots = I
    p, l, u = sla.lu(A)
    assert np.array_equal(p, np.eye(20))
    N = lu_nopivot(A.copy())
    np.testing.assert_allclose(np.tril(N, -1) + np.eye(20), l, atol=1e-14)
    np.testing.assert_allclose(np.triu(N), u, atol=1e-12)


def test_pivot_breakdown_raises():
    from oracle.trees import build_cluster_tree
    ct = build_cluster_tree(np.zeros((3, 3)), 8)
    with pytest.raises(PivotError) as ei:
        lu_nopivot(np.zeros((3, 3)), ct.root)
    assert "cluster 0" in str(ei.value)


@pytest.mark.parametrize("kind", ["lr", "chol"])
def test_probe_residual_cfg1(kind):
    eps = 1e-4
    P = _prob(3, 32, K.KERNEL_SLP if kind == "lr" else K.KERNEL_SLP_SYM)
    G = build(P, eps)
    G0 = G.clone()
    if kind == "lr":
        F, fo = lr(G, eps)
    else:
        F, fo, delta = chol_with_restart(G, eps)
        assert delta == 0.0    # sym(G) is SPD: no shift expected
    v = probe_vectors(P.ct.n)[P.perm]
    res = probe_residual(G0, F, v, kind)
    assert res <= 50 * eps, res
    assert fo.min_pivot > 0
