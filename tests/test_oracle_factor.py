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


@pytest.mark.parametrize("kind", ["lr", "chol"])
def test_solve_factor_and_precond_error(kind):
    """solve_factor (block substitution through the cluster tree) equals
    numpy.linalg.solve with the dense operator apply_factor(F, part, I) for
    every part; the power-iteration preconditioner error
    converges to numpy.linalg.norm(I - (F)^{-1} G, 2)."""
    from oracle.factor import apply_factor, precond_error, solve_factor
    from oracle import kernel as Kk
    x, w = sphere_points(2)
    P = Problem(x, w, 8, 2.0, kernel=Kk.KERNEL_SLP if kind == "lr" else Kk.KERNEL_SLP_SYM)
    G = build(P, 1e-3)
    F, _ = (lr if kind == "lr" else chol)(G.clone(), 1e-3)
    n = P.ct.n
    rng = np.random.default_rng(7)
    V = rng.standard_normal((n, 3))
    parts = ["L", "R", "LT", "RT"] if kind == "lr" else ["Lc", "LcT"]
    for part in parts:
        M = apply_factor(F, part, np.eye(n))
        ref = np.linalg.solve(M, V)
        got = solve_factor(F, part, V.copy())
        assert np.linalg.norm(got - ref) <= 1e-10 * np.linalg.norm(ref), part
    Gd = G.to_dense()
    if kind == "lr":
        Fd = apply_factor(F, "L", apply_factor(F, "R", np.eye(n)))
    else:
        Fd = apply_factor(F, "Lc", apply_factor(F, "LcT", np.eye(n)))
    E = np.eye(n) - np.linalg.solve(Fd, Gd)
    exact = np.linalg.norm(E, 2)
    est = precond_error(G, F, kind, iters=200)
    assert abs(est - exact) <= 1e-3 * exact, (est, exact)
    assert 1e-6 < exact < 1.0


def test_dlp_kernel_pins():
    """Double-layer matrix K + I/2 (reading R20): entries by
    hand, unit diagonal 1/2, and the Gauss integral of the closed polyhedral
    sphere: the row sums of K (without the I/2) tend to +1/2 at the O(h) rate
    of the one-point collocation (error halves per refinement)."""
    from oracle import kernel as Kk
    from hm_inputs import sphere_normals
    x = np.array([[0.0, 0.0, 0.0], [0.0, 0.0, 2.0]])
    w = np.array([0.3, 0.7])
    nr = np.array([[0.0, 0.0, 1.0], [0.0, 0.0, -1.0]])
    Kd = Kk.dense_matrix(x, w, kernel=Kk.KERNEL_DLP, nrm=nr)
    # K_01 = w_1 ((x_1 - x_0) . n_1) / (4 pi 2^3) = 0.7 * (-2) / (32 pi)
    assert Kd[0, 1] == pytest.approx(0.7 * -2.0 / (32 * np.pi), rel=1e-15)
    assert Kd[1, 0] == pytest.approx(0.3 * -2.0 / (32 * np.pi), rel=1e-15)
    assert Kd[0, 0] == Kd[1, 1] == 0.5
    devs = []
    for L in (2, 3, 4):
        xs, ws = sphere_points(L)
        Kd = Kk.dense_matrix(xs, ws, kernel=Kk.KERNEL_DLP, nrm=sphere_normals(L))
        devs.append(np.abs(Kd.sum(1) - 0.5 - 0.5).max())
    assert devs[2] < 0.01 and devs[1] < 0.6 * devs[0] and devs[2] < 0.6 * devs[1], devs


def test_lr_of_dlp_probe_residual():
    """H-LR with accumulated updates of the double-layer matrix K (the paper's
    second test matrix, Fig. 11 right): probe residual of
    L R ~ K within 50 eps (reading #21), preconditioner error finite."""
    from oracle import kernel as Kk
    from oracle.factor import precond_error
    from hm_inputs import sphere_normals
    x, w = sphere_points(3)
    P = Problem(x, w, 32, 2.0, kernel=Kk.KERNEL_DLP, nrm=sphere_normals(3))
    G = build(P, 1e-4)
    F, fo = lr(G.clone(), 1e-4)
    v = probe_vectors(P.ct.n)[P.perm]
    assert probe_residual(G, F, v, "lr") <= 50 * 1e-4
    err = precond_error(G, F, "lr", iters=20)
    assert 0 < err < 0.1, err
