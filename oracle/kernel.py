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
KERNEL_DLP = 2   # double layer K + 1/2 I, needs unit normals


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


def dlp_entries(x, w, nrm, rows, cols):
    """Dense block of the double-layer matrix K + 1/2 I (PAPER.md P:L1583-1585,
    "the double layer potential operator (plus 1/2 times the identity)"),
    collocation at the centroids, one-point quadrature on panel j:

        K_ij = w_j ((x_j - x_i) . n_j) / (4 pi |x_i - x_j|^3),  i != j
        K_ii = 1/2      (the flat panel's own DLP integral vanishes: x_i lies
                         in its plane; plus 1/2 from the identity)

    n_j = outward unit normal.  Sign (reading R20): the kernel is
    -dG/dn_y for G = 1/(4 pi |x-y|), so that the Gauss integral of a closed
    surface gives K 1 ~ +1/2 and K + 1/2 I ~ I on constants: the second-kind
    operator the paper factorizes is invertible (the other sign makes
    1/2 I + K singular on constants).  Evaluated as
    (w_j * dot) / ((4.0*pi*r2) * r) with dot = dx*nx + dy*ny + dz*nz,
    d = x_j - x_i, r2 = dx*dx + dy*dy + dz*dz, r = sqrt(r2), in that order."""
    rows = np.asarray(rows)
    cols = np.asarray(cols)
    xi = x[rows]
    xj = x[cols]
    nj = nrm[cols]
    dx = xj[:, 0][None, :] - xi[:, 0][:, None]
    dy = xj[:, 1][None, :] - xi[:, 1][:, None]
    dz = xj[:, 2][None, :] - xi[:, 2][:, None]
    dot = dx * nj[:, 0][None, :] + dy * nj[:, 1][None, :] + dz * nj[:, 2][None, :]
    r2 = dx * dx + dy * dy + dz * dz
    r = np.sqrt(r2)
    same = rows[:, None] == cols[None, :]
    with np.errstate(divide="ignore", invalid="ignore"):
        g = (w[cols][None, :] * dot) / ((4.0 * np.pi * r2) * r)
    if same.any():
        g[same] = 0.5
    return g


def entries(x, w, rows, cols, kernel=KERNEL_SLP, nrm=None):
    if kernel == KERNEL_SLP:
        return slp_entries(x, w, rows, cols)
    if kernel == KERNEL_SLP_SYM:
        return 0.5 * (slp_entries(x, w, rows, cols) + slp_entries(x, w, cols, rows).T)
    if kernel == KERNEL_DLP:
        if nrm is None:
            raise ValueError("the double-layer kernel needs unit normals")
        return dlp_entries(x, w, nrm, rows, cols)
    raise ValueError(f"unknown kernel {kernel}")


def dense_matrix(x, w, perm=None, kernel=KERNEL_SLP, nrm=None):
    """Full dense matrix; in tree order if perm (tree pos -> original) given."""
    idx = np.arange(len(x)) if perm is None else np.asarray(perm)
    return entries(x, w, idx, idx, kernel, nrm)
