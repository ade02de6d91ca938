"""Refined-icosahedron surface mesh and seeded probe vectors (inputs only).

SURVEY.md §8(c) O1: base icosahedron with vertices (±1,±φ,0), (0,±1,±φ),
(±φ,0,±1) normalised; each refinement splits every triangle 4-way at edge
midpoints that are re-normalised onto the unit sphere; child order
(a,ab,ca), (b,bc,ab), (c,ca,bc), (ab,bc,ca).  Collocation point = flat
centroid (p0+p1+p2)/3, weight = flat area |(p1-p0)x(p2-p0)|/2.
"""
from __future__ import annotations

import numpy as np

_PHI = (1.0 + 5.0 ** 0.5) / 2.0


def _base_icosahedron():
    p = _PHI
    v = np.array(
        [
            [-1, p, 0], [1, p, 0], [-1, -p, 0], [1, -p, 0],
            [0, -1, p], [0, 1, p], [0, -1, -p], [0, 1, -p],
            [p, 0, -1], [p, 0, 1], [-p, 0, -1], [-p, 0, 1],
        ],
        dtype=np.float64,
    )
    v /= np.linalg.norm(v, axis=1)[:, None]
    f = np.array(
        [
            [0, 11, 5], [0, 5, 1], [0, 1, 7], [0, 7, 10], [0, 10, 11],
            [1, 5, 9], [5, 11, 4], [11, 10, 2], [10, 7, 6], [7, 1, 8],
            [3, 9, 4], [3, 4, 2], [3, 2, 6], [3, 6, 8], [3, 8, 9],
            [4, 9, 5], [2, 4, 11], [6, 2, 10], [8, 6, 7], [9, 8, 1],
        ],
        dtype=np.int64,
    )
    return v, f


def icosphere(level: int):
    """Return (vertices (nv,3), faces (n,3)) of the level-`level` refinement."""
    if level < 0:
        raise ValueError("level must be >= 0")
    verts, faces = _base_icosahedron()
    verts = [tuple(x) for x in verts]
    for _ in range(level):
        cache: dict[tuple[int, int], int] = {}

        def mid(i, j):
            key = (i, j) if i < j else (j, i)
            k = cache.get(key)
            if k is None:
                a = np.array(verts[i])
                b = np.array(verts[j])
                m = 0.5 * (a + b)
                m /= np.sqrt(m[0] * m[0] + m[1] * m[1] + m[2] * m[2])
                verts.append(tuple(m))
                k = len(verts) - 1
                cache[key] = k
            return k

        nf = np.empty((4 * len(faces), 3), dtype=np.int64)
        for q, (a, b, c) in enumerate(faces):
            ab, bc, ca = mid(a, b), mid(b, c), mid(c, a)
            nf[4 * q + 0] = (a, ab, ca)
            nf[4 * q + 1] = (b, bc, ab)
            nf[4 * q + 2] = (c, ca, bc)
            nf[4 * q + 3] = (ab, bc, ca)
        faces = nf
    return np.array(verts, dtype=np.float64), np.asarray(faces)


def sphere_points(level: int):
    """Collocation points (n,3) (flat centroids) and weights (n,) (flat areas)."""
    v, f = icosphere(level)
    p0, p1, p2 = v[f[:, 0]], v[f[:, 1]], v[f[:, 2]]
    x = (p0 + p1 + p2) / 3.0
    cr = np.cross(p1 - p0, p2 - p0)
    area = 0.5 * np.sqrt(cr[:, 0] * cr[:, 0] + cr[:, 1] * cr[:, 1] + cr[:, 2] * cr[:, 2])
    return np.ascontiguousarray(x), np.ascontiguousarray(area)


def sphere_normals(level: int):
    """Unit normals (n,3) of the flat triangles, oriented outward
    (n . centroid > 0) -- geometry of the double-layer matrix K (PAPER.md
    P:L1583-1585)."""
    v, f = icosphere(level)
    p0, p1, p2 = v[f[:, 0]], v[f[:, 1]], v[f[:, 2]]
    cr = np.cross(p1 - p0, p2 - p0)
    nrm = cr / np.sqrt(cr[:, 0] * cr[:, 0] + cr[:, 1] * cr[:, 1] + cr[:, 2] * cr[:, 2])[:, None]
    x = (p0 + p1 + p2) / 3.0
    sgn = np.where(np.sum(nrm * x, axis=1) < 0.0, -1.0, 1.0)
    return np.ascontiguousarray(nrm * sgn[:, None])


def random_points(n: int, seed: int):
    """Seeded random points on the unit sphere with random positive weights
    (small structural test inputs: ragged trees, odd n)."""
    rng = np.random.default_rng([1703, 9085, 77, seed])
    x = rng.standard_normal((n, 3))
    x /= np.linalg.norm(x, axis=1)[:, None]
    w = rng.uniform(0.5, 1.5, n) * (4.0 * np.pi / max(n, 1))
    return x, w


def probe_vectors(n: int, count: int = 8):
    """v_j = default_rng([1703, 9085, j]).standard_normal(n),
    in ORIGINAL point order (callers permute into tree order)."""
    return np.stack(
        [np.random.default_rng([1703, 9085, j]).standard_normal(n) for j in range(count)],
        axis=1,
    )
