"""Cluster tree and block tree (§2, Defs 2.1-2.3).

Construction rules are SURVEY.md §8(c) O2 (the paper defers to "standard
algorithms"):
  * cluster: tight bounding box of its points; split the longest axis (ties
    -> lowest axis) at mid = 0.5*(lo+hi); points with x[ax] < mid go to son
    0, the rest to son 1, stable; if a side is empty split by index at
    size//2.  Leaf iff size <= leaf_size.  Binary (§6 assumption P:L1361).
  * block (t,s): admissible leaf iff max(d_t^2, d_s^2) <= eta^2 dist^2
    (BASELINE "max(diam) <= 2*dist"); else inadmissible (dense) leaf iff t or
    s is a cluster leaf (guarantees eq. blocktree_admissible);
    else sons(t) x sons(s), row-major (Def 2.2).
Ids are assigned in breadth-first order, so every level is contiguous and
the sons of a node are consecutive.

Pinned by tests/test_oracle_inputs_trees.py: hand-executed bisection of collinear
points, brute-force classification of every (t,s) pair, partition /
tiling invariants, eq. blocktree_admissible, product-tree membership.
"""
from __future__ import annotations

from collections import deque

import numpy as np

SUB, ADM, DENSE = 0, 1, 2


class Cluster:
    __slots__ = ("id", "start", "size", "level", "sons", "lo", "hi", "parent")

    def __init__(self, start, size, level, lo, hi, parent=None):
        self.id = -1
        self.start = start
        self.size = size
        self.level = level
        self.sons = []
        self.lo = lo
        self.hi = hi
        self.parent = parent

    @property
    def leaf(self):
        return not self.sons

    def __repr__(self):
        return f"C{self.id}[{self.start}:{self.start + self.size}]"


class ClusterTree:
    def __init__(self, root, clusters, perm):
        self.root = root
        self.clusters = clusters  # BFS order, clusters[i].id == i
        self.perm = perm          # tree position -> original index

    @property
    def n(self):
        return self.root.size

    def depth(self):
        return max(c.level for c in self.clusters)

    def leaves(self):
        return [c for c in self.clusters if c.leaf]


def _bbox(pts):
    lo = np.array([pts[:, a].min() for a in range(3)])
    hi = np.array([pts[:, a].max() for a in range(3)])
    return lo, hi


def build_cluster_tree(points, leaf_size):
    """Def 2.1 with the O2 bisection rule."""
    points = np.asarray(points, dtype=np.float64)
    n = len(points)
    if n == 0:
        raise ValueError("empty point set")
    if leaf_size < 1:
        raise ValueError("leaf_size must be >= 1")
    perm = np.arange(n)
    lo, hi = _bbox(points)
    root = Cluster(0, n, 0, lo, hi)
    stack = [root]
    while stack:
        c = stack.pop()
        if c.size <= leaf_size:
            continue
        idx = perm[c.start:c.start + c.size]
        ext = c.hi - c.lo
        ax = 0
        for a in (1, 2):
            if ext[a] > ext[ax]:
                ax = a
        mid = 0.5 * (c.lo[ax] + c.hi[ax])
        mask = points[idx, ax] < mid
        left = idx[mask]
        right = idx[~mask]
        if len(left) == 0 or len(right) == 0:
            left = idx[: c.size // 2]
            right = idx[c.size // 2:]
        perm[c.start:c.start + c.size] = np.concatenate([left, right])
        for off, part in ((0, left), (len(left), right)):
            plo, phi = _bbox(points[part])
            s = Cluster(c.start + off, len(part), c.level + 1, plo, phi, c)
            c.sons.append(s)
        stack.extend(c.sons)
    # breadth-first ids
    clusters = []
    q = deque([root])
    while q:
        c = q.popleft()
        c.id = len(clusters)
        clusters.append(c)
        q.extend(c.sons)
    return ClusterTree(root, clusters, perm)


def diam2(c):
    d = 0.0
    for a in range(3):
        e = c.hi[a] - c.lo[a]
        d = d + e * e
    return d


def dist2(t, s):
    d = 0.0
    for a in range(3):
        g = max(0.0, s.lo[a] - t.hi[a], t.lo[a] - s.hi[a])
        d = d + g * g
    return d


def admissible(t, s, eta):
    return max(diam2(t), diam2(s)) <= (eta * eta) * dist2(t, s)


class Block:
    __slots__ = ("id", "t", "s", "kind", "sons", "level", "parent")

    def __init__(self, t, s, kind, level, parent=None):
        self.id = -1
        self.t = t
        self.s = s
        self.kind = kind
        self.sons = []
        self.level = level
        self.parent = parent

    @property
    def leaf(self):
        return self.kind != SUB

    def son(self, i, j):
        """son (t_i, s_j), i,j = son indices of t and s (row-major)."""
        return self.sons[i * len(self.s.sons) + j]

    def __repr__(self):
        k = "SAD"[self.kind]
        return f"B{self.id}{k}({self.t.id},{self.s.id})"


class BlockTree:
    def __init__(self, root, blocks, rows, cols, eta):
        self.root = root
        self.blocks = blocks   # BFS order
        self.rows = rows       # ClusterTree
        self.cols = cols
        self.eta = eta
        self._index = {(b.t.id, b.s.id): b for b in blocks}

    def find(self, t, s):
        """Block (t,s) if it is a node of the tree, else None."""
        return self._index.get((t.id, s.id))

    def leaves(self):
        return [b for b in self.blocks if b.leaf]

    def depth(self):
        return max(b.level for b in self.blocks)

    def sparsity(self):
        """C_sp of eqs. blocktree_rowsparse/colsparse."""
        rc, cc = {}, {}
        for b in self.blocks:
            rc[b.t.id] = rc.get(b.t.id, 0) + 1
            cc[b.s.id] = cc.get(b.s.id, 0) + 1
        return max(rc.values()), max(cc.values())


def build_block_tree(rows, cols, eta):
    """Def 2.2 with the O2 admissibility rule."""
    root = Block(rows.root, cols.root, SUB, 0)
    blocks = []
    q = deque([root])
    while q:
        b = q.popleft()
        b.id = len(blocks)
        blocks.append(b)
        t, s = b.t, b.s
        if admissible(t, s, eta):
            b.kind = ADM
        elif t.leaf or s.leaf:
            b.kind = DENSE
        else:
            b.kind = SUB
            for ts in t.sons:
                for ss in s.sons:
                    sb = Block(ts, ss, SUB, b.level + 1, b)
                    b.sons.append(sb)
            q.extend(b.sons)
    return BlockTree(root, blocks, rows, cols, eta)


def tree_arrays(ct: ClusterTree, bt: BlockTree):
    """Flat arrays (the hm_host_desc schema of include/hm.h)."""
    C = ct.clusters
    cl = dict(
        cl_start=np.array([c.start for c in C], np.int32),
        cl_size=np.array([c.size for c in C], np.int32),
        cl_son0=np.array([c.sons[0].id if c.sons else -1 for c in C], np.int32),
        cl_nsons=np.array([len(c.sons) for c in C], np.int32),
        cl_level=np.array([c.level for c in C], np.int32),
        cl_bbox=np.array([np.concatenate([c.lo, c.hi]) for c in C], np.float64),
    )
    B = bt.blocks
    bl = dict(
        bl_row=np.array([b.t.id for b in B], np.int32),
        bl_col=np.array([b.s.id for b in B], np.int32),
        bl_kind=np.array([b.kind for b in B], np.int32),
        bl_son0=np.array([b.sons[0].id if b.sons else -1 for b in B], np.int32),
        bl_nsons=np.array([len(b.sons) for b in B], np.int32),
    )
    cl.update(bl)
    cl["perm"] = np.asarray(ct.perm, np.int64)
    return cl
