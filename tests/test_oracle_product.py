"""Pins for the H-matrix product schedules S0 / S1 / S2 (§4-5).

  * eps = 0 on tiny n: Z + alpha X Y equals the dense product to 1e-12
    (north-star check 1) for all three schedules; the n=320/leaf-8 case hits
    every Fig. 5 branch and every reachable Fig. 7 branch incl. nested
    virtual recursion.
  * call-tree correspondence: addproduct calls == product-tree nodes
    (P:L1195-1197); S2 updates each Z leaf exactly once.
  * content conservation of split at eps = 0 (sum of terms, no subtraction).
  * truncation counts: S2 < S0 and S2 < S1.
  * eps = 1e-4 at n = 1280: S0/S1/S2 agree within the eps bound; relative
    spectral error "well below 1e-4" as a soft gate.
"""
import numpy as np
import pytest

from hm_inputs import random_points, sphere_points
from oracle.hmatrix import Problem, build
from oracle.lowrank import TruncCtx
from oracle.product import (S2, Acc2, addmul_s0, addmul_s1, addmul_s2, evaluate,
                            product_tree_nodes)
from oracle.trees import ADM, DENSE

SCHEDULES = {"S0": addmul_s0, "S1": addmul_s1, "S2": addmul_s2}


def _problem(L, leaf):
    x, w = sphere_points(L)
    return Problem(x, w, leaf, 2.0)


@pytest.fixture(scope="module")
def tiny320():
    P = _problem(2, 8)
    return P, build(P, 0.0)


@pytest.mark.parametrize("name", ["S0", "S1", "S2"])
@pytest.mark.parametrize("alpha", [1.0, -0.5])
def test_eps0_equals_dense(tiny320, name, alpha):
    P, G = tiny320
    Gd = G.to_dense()
    Z, ctx, st = SCHEDULES[name](alpha, G.clone(), G.clone(), G.clone(), 0.0)
    ref = Gd + alpha * Gd @ Gd
    assert np.linalg.norm(Z.to_dense() - ref) <= 1e-12 * np.linalg.norm(ref)
    assert st.addproduct == len(product_tree_nodes(P.bt, P.bt))


def test_eps0_random_points_distinct_xyz():
    """X, Y, Z different matrices (kernel matrix, its transpose-scaled copy, zero)."""
    x, w = random_points(200, 11)
    P = Problem(x, w, 6, 2.0)
    X = build(P, 0.0)
    Y = X.clone()
    for k in Y.A:
        Y.A[k] = 2.0 * Y.A[k]
    for k in Y.N:
        Y.N[k] = Y.N[k] + 1.0
    Z = X.clone()
    for k in Z.N:
        Z.N[k][:] = 0.0
    for k in Z.A:
        Z.A[k] = Z.A[k][:, :0]
        Z.B[k] = Z.B[k][:, :0]
    Xd, Yd = X.to_dense(), Y.to_dense()
    out, _, _ = addmul_s2(0.3, X, Y, Z, 0.0)
    ref = 0.3 * Xd @ Yd
    assert np.linalg.norm(out.to_dense() - ref) <= 1e-12 * np.linalg.norm(ref)


def test_branch_coverage_and_leaf_updates(tiny320):
    P, G = tiny320
    Z, ctx, st = addmul_s2(1.0, G.clone(), G.clone(), G.clone(), 0.0)
    assert all(c > 0 for c in st.branch[:6]), st.branch
    for br in ("i_adm", "i_virtual", "ii_dense", "iv_sub", "v_adm", "v_virtual"):
        assert st.flush_branch.get(br, 0) > 0, (br, st.flush_branch)
    assert "iii_sub" not in st.flush_branch   # unreachable in hm_addmul
    leaves = [b.id for b in P.bt.leaves()]
    assert sorted(st.leaf_updates) == sorted(leaves)
    assert set(st.leaf_updates.values()) == {1}


def test_split_conserves_content(tiny320):
    """content(acc) = dense(base)+sum terms + sum_pending alpha X|ts Y|sr is
    conserved by split at eps = 0; sums only, no subtraction."""
    P, G = tiny320
    Gd = G.to_dense()
    alg = S2(G, G, TruncCtx(0.0))
    root = P.bt.root
    acc = Acc2(root.t, root.s)
    alg.addproduct(acc, 1.0, root, root)

    def content(a):
        C = a.content_lowrank()
        for alpha, bx, by, _X, _Y in a.pending:
            X = Gd[bx.t.start:bx.t.start + bx.t.size, bx.s.start:bx.s.start + bx.s.size]
            Y = Gd[by.t.start:by.t.start + by.t.size, by.s.start:by.s.start + by.s.size]
            C = C + alpha * X @ Y
        return C

    level = [acc]
    for depth in range(3):
        nxt = []
        for a in level:
            if not a.pending:
                continue
            before = content(a)
            grid = alg.split(a, (a.t.id, a.r.id))
            after = np.block([[content(s) for s in row] for row in grid])
            np.testing.assert_allclose(after, before, atol=1e-12 * np.abs(before).max())
            nxt += [s for row in grid for s in row]
        level = nxt


def test_evaluate_factorizes_product(tiny320):
    """Every Fig. 5 branch returns an exact factorization of alpha X|ts Y|sr."""
    P, G = tiny320
    Gd = G.to_dense()
    seen = set()
    for bx in P.bt.blocks:
        for by in P.bt.blocks:
            if by.t is not bx.s:
                continue
            ev = evaluate(-1.5, bx, by, G, G)
            if ev is None:
                continue
            key = (bx.kind, by.kind, bx.t.size <= bx.s.size, by.s.size <= by.t.size)
            if key in seen:
                continue
            seen.add(key)
            X = Gd[bx.t.start:bx.t.start + bx.t.size, bx.s.start:bx.s.start + bx.s.size]
            Y = Gd[by.t.start:by.t.start + by.t.size, by.s.start:by.s.start + by.s.size]
            ref = -1.5 * X @ Y
            np.testing.assert_allclose(ev[0] @ ev[1].T, ref, atol=1e-13 * (1 + np.abs(ref).max()))
    assert len(seen) >= 6


@pytest.fixture(scope="module")
def cfg1():
    P = _problem(3, 32)
    G = build(P, 1e-4)
    out = {}
    for name, f in SCHEDULES.items():
        Z, ctx, st = f(1.0, G.clone(), G.clone(), G.clone(), 1e-4)
        out[name] = (Z.to_dense(), ctx, st)
    return P, G, out


def test_truncation_counts(cfg1):
    P, G, out = cfg1
    c0, c1, c2 = (out[k][1].count for k in ("S0", "S1", "S2"))
    assert c2 < c0 and c2 < c1
    assert c2 * 5 < c0


def test_schedules_agree_within_eps(cfg1):
    P, G, out = cfg1
    Gd = G.to_dense()
    ref = Gd + Gd @ Gd
    nref = np.linalg.norm(ref)
    depth = P.bt.depth()
    bound = 2 * (depth + 2) * 1e-4 * nref
    for a in out:
        for b in out:
            assert np.linalg.norm(out[a][0] - out[b][0]) <= bound
    for a in out:
        spec = np.linalg.norm(out[a][0] - ref, 2) / np.linalg.norm(ref, 2)
        assert spec <= 1e-4, (a, spec)
