"""Seeded, synthetic input generators shared by the oracle and the CUDA path.

This module holds NONE of the method's arithmetic (no trees, no kernel
matrix, no truncation): only the geometry of the workload and the random
probe vectors.  It is the single place both sides may import.

Workload recipe (BASELINE.json configs):
  * refined icosahedron on the unit sphere, level L -> n = 20 * 4**L
    triangles (L = 3..7 -> 1280 ... 327680),
  * collocation point = flat triangle centroid (not re-projected),
  * weight = flat triangle area.
The paper (§7) uses a refined double pyramid; the
icosahedron is BASELINE.json's stand-in.
"""
from .mesh import icosphere, sphere_normals, sphere_points, probe_vectors, random_points

__all__ = ["icosphere", "sphere_normals", "sphere_points", "probe_vectors", "random_points"]
