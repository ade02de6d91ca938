"""Per-block summaries of an H-matrix for the full-size golden files
(TEST INFRASTRUCTURE: only tests/, scripts/make_golden.py, smoke() and
bench.py's CPU legs use it; the CUDA path never imports oracle/).

A golden file cannot hold a 460 MB H-matrix, so each leaf block b = (t, r)
is summarised by
  * its rank (admissible leaves) and exact Frobenius norm ||Z_b||_F (via QR
    of the factors, never the Gram expansion),
  * a two-sided Gaussian sketch S_b = Omega_L[t]^T Z_b Omega_R[r] (k x k,
    k = 4; 2 for the n = 327680 golden), Omega_L, Omega_R = n x k standard
    normal panels in tree order with fixed
    seeds (1703, 9085, 97) / (1703, 9085, 96).
For a difference D_b of two results, E ||Omega_L^T D_b Omega_R||_F^2 =
k^2 ||D_b||_F^2 (independent standard normal panels), so
||S_b(Z_gpu) - S_b(Z_oracle)||_F / k estimates the per-block Frobenius
difference of the north star's parity rule without storing the block.
Sketches are linear in Z_b: summaries of the two results are compared
directly, block by block, for EVERY leaf.
"""
from __future__ import annotations

import numpy as np

ADM, DENSE = 1, 2
SKETCH_K = 4


def sketch_panels(n, k=SKETCH_K):
    """Omega_L, Omega_R (n x k, tree order)."""
    oml = np.random.default_rng([1703, 9085, 97]).standard_normal((n, k))
    omr = np.random.default_rng([1703, 9085, 96]).standard_normal((n, k))
    return oml, omr


def lowrank_fro(A, B):
    """||A B^T||_F via QR of both factors."""
    if A.shape[1] == 0:
        return 0.0
    _, Ra = np.linalg.qr(A)
    _, Rb = np.linalg.qr(B)
    return float(np.linalg.norm(Ra @ Rb.T))


def summarise_payloads(n, leaves, payload, k=SKETCH_K):
    """leaves: list of (block id, kind, row0, m, col0, n_b) over all leaves;
    payload(bid) -> ('adm', A, B) | ('dense', N).  Returns a dict of arrays:
    leaf_ids, ranks (-1 for dense), fro, sk (nleaves x 4 x 4)."""
    oml, omr = sketch_panels(n, k)
    nl = len(leaves)
    ids = np.zeros(nl, np.int64)
    ranks = np.full(nl, -1, np.int32)
    fro = np.zeros(nl)
    sk = np.zeros((nl, k, k))
    for i, (bid, kind, r0, m, c0, nb) in enumerate(leaves):
        ids[i] = bid
        L = oml[r0:r0 + m]
        R = omr[c0:c0 + nb]
        v = payload(bid)
        if v[0] == "adm":
            A, B = v[1], v[2]
            ranks[i] = A.shape[1]
            fro[i] = lowrank_fro(A, B)
            sk[i] = (L.T @ A) @ (B.T @ R)
        else:
            N = v[1]
            fro[i] = float(np.linalg.norm(N))
            sk[i] = L.T @ (N @ R)
    return dict(leaf_ids=ids, ranks=ranks, fro=fro, sk=sk)


def summarise_hmatrix(h, k=SKETCH_K):
    """Summary of an oracle HMatrix (oracle/hmatrix.py)."""
    leaves = []
    for b in sorted(h.bt.leaves(), key=lambda b: b.id):
        leaves.append((b.id, b.kind, b.t.start, b.t.size, b.s.start, b.s.size))

    def payload(bid):
        if bid in h.A:
            return ("adm", h.A[bid], h.B[bid])
        return ("dense", h.N[bid])

    return summarise_payloads(h.n, leaves, payload, k)


def summarise_desc(d, k=SKETCH_K):
    """Summary of an hm_host_desc dict (include/hm.h schema: what hm_export
    returns, or oracle.hmatrix.export)."""
    cs, cz = d["cl_start"], d["cl_size"]
    leaves = []
    for b in range(len(d["bl_row"])):
        kind = int(d["bl_kind"][b])
        if kind == 0:
            continue
        t, s = int(d["bl_row"][b]), int(d["bl_col"][b])
        leaves.append((b, kind, int(cs[t]), int(cz[t]), int(cs[s]), int(cz[s])))

    def payload(b):
        t, s = int(d["bl_row"][b]), int(d["bl_col"][b])
        m, nb = int(cz[t]), int(cz[s])
        o = int(d["bl_off"][b])
        if int(d["bl_kind"][b]) == ADM:
            k = int(d["bl_rank"][b])
            A = d["factors"][o:o + m * k].reshape((m, k), order="F")
            B = d["factors"][o + m * k:o + (m + nb) * k].reshape((nb, k), order="F")
            return ("adm", A, B)
        return ("dense", d["dense"][o:o + m * nb].reshape((m, nb), order="F"))

    return summarise_payloads(int(d["n"]), leaves, payload, k)


def compare_summaries(got, ref, tol, allowed=frozenset(), eps_bound=None):
    """North-star parity on summaries: identical ranks except on `allowed`
    blocks (near-threshold truncations), and per-block difference estimate
    ||S_got - S_ref||_F / 4 <= tol * max(||Z_ref,b||_F, 1e-12 ||Z_ref||_F)
    (allowed blocks whose rank flipped: <= eps_bound * the same denominator).
    Returns a report."""
    assert np.array_equal(got["leaf_ids"], ref["leaf_ids"]), "different leaf sets"
    znorm = float(np.sqrt(np.sum(ref["fro"] ** 2)))
    den = np.maximum(ref["fro"], 1e-12 * znorm)
    diff = np.sqrt(np.sum((got["sk"] - ref["sk"]) ** 2, axis=(1, 2))) / ref["sk"].shape[1]
    rel = diff / den
    ids = ref["leaf_ids"]
    flipped = got["ranks"] != ref["ranks"]
    mism = [int(ids[i]) for i in np.nonzero(flipped)[0]]
    # only a near-flagged block whose rank actually flipped gets the eps bound;
    # every other block (incl. near-flagged ones with equal rank) is strict
    in_allowed = np.array([int(b) in allowed for b in ids], bool) & flipped
    strict = ~in_allowed
    worst = float(rel[strict].max()) if strict.any() else 0.0
    worst_b = int(ids[strict][np.argmax(rel[strict])]) if strict.any() else None
    worst_allowed = float(rel[in_allowed].max()) if in_allowed.any() else 0.0
    fro_rel = np.abs(got["fro"] - ref["fro"]) / den
    return dict(rank_mismatch=mism, unexplained_mismatch=[b for b in mism if b not in allowed],
                worst=worst, worst_block=worst_b, worst_allowed=worst_allowed,
                worst_fro=float(fro_rel[strict].max()) if strict.any() else 0.0,
                nleaves=len(ids), znorm=znorm, tol=tol, eps_bound=eps_bound,
                ok=(not [b for b in mism if b not in allowed]) and worst <= tol and
                   (eps_bound is None or worst_allowed <= eps_bound))


def near_blocks(d_or_tree, near_tags):
    """Leaf block ids inside the (t, r) cluster pairs of near-threshold
    truncations (north star exemption).  d_or_tree: hm_host_desc dict;
    near_tags: iterable of (t_cluster_id, r_cluster_id)."""
    d = d_or_tree
    cs, cz = d["cl_start"], d["cl_size"]
    rngs = [(int(cs[t]), int(cs[t]) + int(cz[t]), int(cs[r]), int(cs[r]) + int(cz[r])) for t, r in near_tags]
    out = set()
    if not rngs:
        return out
    for b in range(len(d["bl_row"])):
        if int(d["bl_kind"][b]) == 0:
            continue
        t, s = int(d["bl_row"][b]), int(d["bl_col"][b])
        t0, t1, s0, s1 = int(cs[t]), int(cs[t]) + int(cz[t]), int(cs[s]), int(cs[s]) + int(cz[s])
        for a0, a1, b0, b1 in rngs:
            if a0 <= t0 and t1 <= a1 and b0 <= s0 and s1 <= b1:
                out.add(b)
                break
    return out
