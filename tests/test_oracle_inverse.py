"""Pins of oracle/inverse.py (Fig. 8: H-matrix inversion with
accumulated updates)."""
import numpy as np
import pytest

from hm_inputs import sphere_points
from oracle.hmatrix import Problem, build
from oracle.inverse import _zero_subtree, inverse_precond_error, invert
from oracle.lowrank import TruncCtx


@pytest.mark.parametrize("L,leaf", [(1, 4), (2, 8)])
def test_invert_exact_at_eps0(L, leaf):
    """eps = 0: no truncation drops anything, so the result is the exact
    inverse: G_dense @ inv_dense = I to 1e-10 (condition ~2 at these sizes)."""
    x, w = sphere_points(L)
    P = Problem(x, w, leaf, 2.0)
    G = build(P, 0.0)
    Gd = G.to_dense()
    Gi, inv = invert(G.clone(), 0.0)
    Id = Gd @ Gi.to_dense()
    assert np.linalg.norm(Id - np.eye(P.ct.n)) <= 1e-10 * np.sqrt(P.ct.n)
    assert inv.leaf_inverses == sum(1 for c in P.ct.leaves())


def test_invert_block_diagonal():
    """Off-diagonal blocks zero: the inverse is blockwise (the two halves
    never interact: H12 = H21 = 0, S = G22)."""
    x, w = sphere_points(2)
    P = Problem(x, w, 8, 2.0)
    G = build(P, 1e-6)
    root = P.bt.root
    t1, t2 = root.t.sons
    _zero_subtree(G, P.bt.find(t1, t2))
    _zero_subtree(G, P.bt.find(t2, t1))
    Gd = G.to_dense()
    Gi, _ = invert(G.clone(), 0.0)
    n1 = t1.size
    ref1 = np.linalg.inv(Gd[:n1, :n1])
    ref2 = np.linalg.inv(Gd[n1:, n1:])
    D = Gi.to_dense()
    assert np.linalg.norm(D[:n1, :n1] - ref1) <= 1e-10 * np.linalg.norm(ref1)
    assert np.linalg.norm(D[n1:, n1:] - ref2) <= 1e-10 * np.linalg.norm(ref2)
    assert np.abs(D[:n1, n1:]).max() == 0.0 and np.abs(D[n1:, :n1]).max() == 0.0


def test_invert_precond_error_eps():
    """eps = 1e-4, n = 1280: the power-iteration preconditioner error
     agrees with the exact ||I - G~^{-1} G||_2 and is of the
    order the paper reports for the single-layer matrix at small n (6e-4,
    P:L1630-1632; different matrix: a soft range, not a value)."""
    x, w = sphere_points(3)
    P = Problem(x, w, 32, 2.0)
    G = build(P, 1e-4)
    ctx = TruncCtx(1e-4)
    Gi, _ = invert(G.clone(), 1e-4, ctx)
    E = np.eye(P.ct.n) - Gi.to_dense() @ G.to_dense()
    exact = np.linalg.norm(E, 2)
    est = inverse_precond_error(G, Gi, iters=100)
    assert abs(est - exact) <= 1e-3 * exact, (est, exact)
    assert 1e-6 < exact < 1e-2, exact
    assert ctx.count > 0
