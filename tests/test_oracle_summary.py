"""Pins of oracle/summary.py (golden-file summaries): the two-sided sketch
estimates per-block Frobenius differences (E ||Om_L^T D Om_R||^2 = k^2 ||D||^2
for independent standard normal panels), summaries of an HMatrix and of its
exported host description agree exactly, a 1e-8 perturbation of one block
is caught at the 1e-9 tolerance, and near-threshold exemptions cover exactly
the leaves inside the flagged (t, r) block."""
import numpy as np

from hm_inputs import sphere_points
from oracle.hmatrix import Problem, build, export
from oracle.summary import (compare_summaries, lowrank_fro, near_blocks, sketch_panels, summarise_desc,
                            summarise_hmatrix)


def test_sketch_estimates_frobenius():
    rng = np.random.default_rng(1)
    n, k = 4000, 4
    ratios = []
    for i in range(400):
        m = int(rng.integers(5, 60))
        D = rng.standard_normal((m, 3)) @ rng.standard_normal((3, m))   # rank 3
        L = rng.standard_normal((m, k))
        R = rng.standard_normal((m, k))
        ratios.append(np.sum((L.T @ D @ R) ** 2) / (k * k * np.sum(D ** 2)))
    assert abs(np.mean(ratios) - 1.0) < 0.1
    oml, omr = sketch_panels(n)
    assert oml.shape == (n, 4) and not np.allclose(oml, omr)


def test_lowrank_fro():
    rng = np.random.default_rng(2)
    A, B = rng.standard_normal((50, 6)), rng.standard_normal((40, 6))
    assert abs(lowrank_fro(A, B) - np.linalg.norm(A @ B.T)) <= 1e-12 * np.linalg.norm(A @ B.T)
    assert lowrank_fro(A[:, :0], B[:, :0]) == 0.0


def test_summary_desc_equals_hmatrix_and_detects_perturbation():
    x, w = sphere_points(2)
    P = Problem(x, w, 8, 2.0)
    G = build(P, 1e-4)
    d = export(G)
    s1 = summarise_hmatrix(G)
    s2 = summarise_desc(d)
    for key in ("leaf_ids", "ranks"):
        assert np.array_equal(s1[key], s2[key]), key
    for key in ("fro", "sk"):   # same numbers; only the memory layout (BLAS order) differs
        np.testing.assert_allclose(s1[key], s2[key], rtol=1e-13, atol=1e-15)
    rep = compare_summaries(s2, s1, 1e-9)
    assert rep["ok"] and rep["worst"] <= 1e-13
    # perturb one admissible block by 1e-8 relative: must fail at 1e-9
    H = G.clone()
    bid = next(iter(H.A))
    A = H.A[bid]
    H.A[bid] = A * (1 + 1e-8)
    rep = compare_summaries(summarise_hmatrix(H), s1, 1e-9)
    assert not rep["ok"] and rep["worst_block"] == bid
    # a dense block with a single-entry error of 1e-8 ||N||
    H = G.clone()
    bid = next(iter(H.N))
    H.N[bid][0, 0] += 1e-8 * np.linalg.norm(H.N[bid])
    rep = compare_summaries(summarise_hmatrix(H), s1, 1e-9)
    assert not rep["ok"] and rep["worst_block"] == bid
    # a rank change is reported unless the block is near-flagged
    H = G.clone()
    bid = next(b for b in H.A if H.A[b].shape[1] >= 2)
    H.A[bid] = H.A[bid][:, :-1]
    H.B[bid] = H.B[bid][:, :-1]
    b = P.bt.blocks[bid]
    rep = compare_summaries(summarise_hmatrix(H), s1, 1e-9)
    assert rep["unexplained_mismatch"] == [bid]
    allowed = near_blocks(d, [(b.t.id, b.s.id)])
    rep = compare_summaries(summarise_hmatrix(H), s1, 1e-9, allowed, eps_bound=1.0)
    assert rep["unexplained_mismatch"] == [] and rep["rank_mismatch"] == [bid]


def test_near_blocks_subtree():
    x, w = sphere_points(2)
    P = Problem(x, w, 8, 2.0)
    d = export(build(P, 1e-4))
    root = P.bt.root
    assert len(near_blocks(d, [(root.t.id, root.s.id)])) == len(P.bt.leaves())
    sub = next(b for b in P.bt.blocks if b.kind == 0 and b is not root)
    got = near_blocks(d, [(sub.t.id, sub.s.id)])
    want = set()
    st = [sub]
    while st:
        c = st.pop()
        if c.kind == 0:
            st.extend(c.sons)
        else:
            want.add(c.id)
    assert got == want
