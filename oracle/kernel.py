"""Kernel matrix entries of the synthetic BEM-like workload.

BASELINE.json configs: G_ij = area_j / (4*pi*|x_i - x_j|) for i != j and
G_ii = sqrt(area_i/pi)/2 (exact self-integral of 1/(4 pi r) over a disk of
area area_i).  Config 3 (Cholesky) uses (G + G^T)/2.
The paper's own matrices are Galerkin SLP/DLP via HCA (§7);
this collocation matrix stands in for them.

Pinned by tests/test_oracle_inputs_trees.py (hand-computed entries, symmetry of the
symmetrised variant, diagonal formula).
"""
from __future__ import annotations

import numpy as np

KERNEL_SLP = 0
KERNEL_SLP_SYM = 1


def slp_entries(x, w, rows, cols):
    """Dense block G[rows, cols] of the (non-symmetric) SLP kernel.

    rows/cols are ORIGINAL point indices.  Evaluated as
    w_j / (4.0*pi*sqrt(dx*dx+dy*dy+dz*dz)) in that operation order."""
    rows = np.asarray(rows)
    cols = np.asarray(cols)
    xi = x[rows]
    xj = x[cols]
    dx = xi[:, 0][:, None] - xj[:, 0][None, :]
    dy = xi[:, 1][:, None] - xj[:, 1][None, :]
    dz = xi[:, 2][:, None] - xj[:, 2][None, :]
    r = np.sqrt(dx * dx + dy * dy + dz * dz)
    same = rows[:, None] == cols[None, :]
    with np.errstate(divide="ignore"):
        g = w[cols][None, :] / (4.0 * np.pi * r)
    if same.any():
        ii, jj = np.nonzero(same)
        g[ii, jj] = np.sqrt(w[rows[ii]] / np.pi) / 2.0
    return g


def entries(x, w, rows, cols, kernel=KERNEL_SLP):
    if kernel == KERNEL_SLP:
        return slp_entries(x, w, rows, cols)
    if kernel == KERNEL_SLP_SYM:
        return 0.5 * (slp_entries(x, w, rows, cols) + slp_entries(x, w, cols, rows).T)
    raise ValueError(f"unknown kernel {kernel}")


def dense_matrix(x, w, perm=None, kernel=KERNEL_SLP):
    """Full dense matrix; in tree order if perm (tree pos -> original) given."""
    idx = np.arange(len(x)) if perm is None else np.asarray(perm)
    return entries(x, w, idx, idx, kernel)
