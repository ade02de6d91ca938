"""Pins for the input generator, kernel entries and the trees of the oracle.

Pins (none re-types the oracle's own formula):
  * mesh: n = 20*4^L, Euler characteristic, vertices on the unit sphere,
    total flat area increases towards 4*pi (inscribed polyhedra).
  * kernel: hand-computed entries for 2 points; the diagonal is the exact
    self-integral of 1/(4 pi r) over a disk (closed form by hand, below).
  * cluster tree: hand-executed bisection of collinear points (SPEC example),
    partition invariants (Def 2.1).
  * block tree: brute-force classification of EVERY cluster pair with an
    independent evaluation of the admissibility rule; leaves tile I x J
    exactly once; eq. blocktree_admissible.
  * product tree: eq. product_block by exhaustive triples.
"""
import itertools
import math

import numpy as np
import pytest

from hm_inputs import icosphere, random_points, sphere_points
from oracle import kernel as K
from oracle.product import product_tree_nodes
from oracle.trees import ADM, DENSE, SUB, build_block_tree, build_cluster_tree


@pytest.mark.parametrize("L", [0, 1, 2, 3])
def test_icosphere_counts(L):
    v, f = icosphere(L)
    assert len(f) == 20 * 4 ** L
    # Euler: V - E + F = 2 for a closed triangulated sphere; E = 3F/2
    assert len(v) - 3 * len(f) // 2 + len(f) == 2
    np.testing.assert_allclose(np.linalg.norm(v, axis=1), 1.0, atol=1e-15)


def test_area_converges_to_sphere():
    sums = [sphere_points(L)[1].sum() for L in range(0, 5)]
    assert all(a < b for a, b in zip(sums, sums[1:]))
    assert all(s < 4 * math.pi for s in sums)
    assert abs(sums[-1] - 4 * math.pi) / (4 * math.pi) < 2e-3


def test_kernel_entries_by_hand():
    x = np.array([[0.0, 0.0, 0.0], [3.0, 4.0, 0.0]])
    w = np.array([2.0, 5.0])
    G = K.dense_matrix(x, w)
    # |x0-x1| = 5  ->  G_01 = w_1 / (4 pi 5) = 5/(20 pi) = 1/(4 pi)
    assert G[0, 1] == pytest.approx(1.0 / (4 * math.pi), rel=1e-15)
    assert G[1, 0] == pytest.approx(2.0 / (20 * math.pi), rel=1e-15)
    # disk of area a, radius rho = sqrt(a/pi): int_disk 1/(4 pi r) dA = rho/2
    assert G[0, 0] == pytest.approx(math.sqrt(2.0 / math.pi) / 2, rel=1e-15)
    assert G[1, 1] == pytest.approx(math.sqrt(5.0 / math.pi) / 2, rel=1e-15)
    Gs = K.dense_matrix(x, w, kernel=K.KERNEL_SLP_SYM)
    assert Gs[0, 1] == Gs[1, 0] == pytest.approx(0.5 * (1 / (4 * math.pi) + 1 / (10 * math.pi)))


def test_kernel_blocks_consistent():
    x, w = sphere_points(1)
    G = K.dense_matrix(x, w)
    rows = np.array([3, 7, 11])
    cols = np.array([0, 7, 40, 2])
    np.testing.assert_array_equal(K.entries(x, w, rows, cols), G[np.ix_(rows, cols)])


def test_cluster_tree_collinear_by_hand():
    pts = np.array([[0.0, 0, 0], [1.0, 0, 0], [2.0, 0, 0], [3.0, 0, 0]])
    ct = build_cluster_tree(pts, 1)
    root = ct.root
    assert list(root.lo) == [0, 0, 0] and list(root.hi) == [3, 0, 0]
    # mid = 1.5: {0,1} | {2,3}; then mid 0.5 and 2.5
    assert [len(c.sons) for c in ct.clusters] == [2, 2, 2, 0, 0, 0, 0]
    assert ct.depth() == 2
    assert list(ct.perm) == [0, 1, 2, 3]
    # reversed input order: perm must sort by x
    ct2 = build_cluster_tree(pts[::-1].copy(), 1)
    assert list(ct2.perm) == [3, 2, 1, 0]


def test_cluster_tree_degenerate_and_single():
    ct = build_cluster_tree(np.zeros((1, 3)), 1)
    assert ct.depth() == 0 and ct.root.leaf
    ct = build_cluster_tree(np.zeros((6, 3)), 2)   # zero extent -> index split
    sizes = [c.size for c in ct.clusters]
    assert sizes[:3] == [6, 3, 3]
    with pytest.raises(ValueError):
        build_cluster_tree(np.zeros((0, 3)), 1)


def _check_partition(ct, leaf_size):
    for c in ct.clusters:
        if c.sons:
            assert len(c.sons) == 2
            assert c.sons[0].start == c.start
            assert c.sons[1].start == c.start + c.sons[0].size
            assert c.sons[0].size + c.sons[1].size == c.size
            assert c.size > leaf_size
        else:
            assert c.size <= leaf_size
    assert sorted(ct.perm) == list(range(ct.n))


@pytest.mark.parametrize("n,leaf,seed", [(37, 3, 0), (100, 8, 1), (211, 16, 2), (64, 1, 3)])
def test_trees_bruteforce(n, leaf, seed):
    x, _ = random_points(n, seed)
    ct = build_cluster_tree(x, leaf)
    _check_partition(ct, leaf)
    # bbox of every cluster is tight
    for c in ct.clusters:
        p = x[ct.perm[c.start:c.start + c.size]]
        np.testing.assert_array_equal(c.lo, p.min(axis=0))
        np.testing.assert_array_equal(c.hi, p.max(axis=0))
    eta = 2.0
    bt = build_block_tree(ct, ct, eta)

    def adm_indep(t, s):
        # independent evaluation with numpy vector ops
        dt = np.sum((t.hi - t.lo) ** 2)
        ds = np.sum((s.hi - s.lo) ** 2)
        gap = np.maximum(0.0, np.maximum(s.lo - t.hi, t.lo - s.hi))
        return max(dt, ds) <= eta ** 2 * np.sum(gap ** 2)

    cover = np.zeros((n, n), dtype=np.int32)
    for b in bt.blocks:
        t, s = b.t, b.s
        a = adm_indep(t, s)
        if b.kind == ADM:
            assert a
        elif b.kind == DENSE:
            assert not a and (t.leaf or s.leaf)
        else:
            assert not a and not t.leaf and not s.leaf
            assert [(c.t.id, c.s.id) for c in b.sons] == [(p.id, q.id) for p in t.sons for q in s.sons]
        if b.leaf:
            cover[t.start:t.start + t.size, s.start:s.start + s.size] += 1
        if b.kind == DENSE:   # eq. blocktree_admissible
            assert t.leaf or s.leaf
    assert (cover == 1).all()
    # every pair reachable from the root by the rule appears exactly once
    ids = {(b.t.id, b.s.id) for b in bt.blocks}
    assert len(ids) == len(bt.blocks)
    # BFS order: levels non-decreasing, sons consecutive
    lv = [b.level for b in bt.blocks]
    assert lv == sorted(lv)
    for b in bt.blocks:
        if b.sons:
            assert [c.id for c in b.sons] == list(range(b.sons[0].id, b.sons[0].id + len(b.sons)))


@pytest.mark.parametrize("n,leaf,seed", [(24, 2, 5), (40, 3, 6)])
def test_product_tree_membership(n, leaf, seed):
    """eq. (product_block): (t,s,r) in T_IxJxK <=> (t,s) in T_IxJ and (s,r) in T_JxK."""
    x, _ = random_points(n, seed)
    ct = build_cluster_tree(x, leaf)
    bt = build_block_tree(ct, ct, 2.0)
    nodes = set(product_tree_nodes(bt, bt))
    pairs = {(b.t.id, b.s.id) for b in bt.blocks}
    C = [c.id for c in ct.clusters]
    brute = {(t, s, r) for t, s, r in itertools.product(C, C, C) if (t, s) in pairs and (s, r) in pairs}
    assert nodes == brute


def test_config1_structure():
    """Shapes quoted for config 1 in SURVEY §8 (structure only, from the rules)."""
    x, w = sphere_points(3)
    ct = build_cluster_tree(x, 32)
    bt = build_block_tree(ct, ct, 2.0)
    assert len(ct.clusters) == 103
    assert len(bt.blocks) == 1837
    assert sum(b.kind == ADM for b in bt.blocks) == 918
    assert sum(b.kind == DENSE for b in bt.blocks) == 460
