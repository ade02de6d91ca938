"""Comparison helpers for GPU <-> oracle parity (test infrastructure)."""
from __future__ import annotations

import numpy as np

ADM, DENSE = 1, 2


def leaf_payloads(d):
    """dict block id -> ('adm', A, B) | ('dense', N) from an hm_host_desc dict."""
    out = {}
    cs, cz = d["cl_start"], d["cl_size"]
    for b in range(len(d["bl_row"])):
        kind = int(d["bl_kind"][b])
        if kind == 0:
            continue
        m = int(cz[d["bl_row"][b]])
        n = int(cz[d["bl_col"][b]])
        o = int(d["bl_off"][b])
        if kind == ADM:
            k = int(d["bl_rank"][b])
            A = d["factors"][o:o + m * k].reshape((m, k), order="F")
            B = d["factors"][o + m * k:o + (m + n) * k].reshape((n, k), order="F")
            out[b] = ("adm", A, B)
        else:
            out[b] = ("dense", d["dense"][o:o + m * n].reshape((m, n), order="F"))
    return out


def lowrank_diff(Ag, Bg, Ao, Bo):
    """||Ag Bg^T - Ao Bo^T||_F via QR of the stacks (never the Gram expansion)."""
    A = np.hstack([Ag, -Ao])
    B = np.hstack([Bg, Bo])
    if A.shape[1] == 0:
        return 0.0
    _, Ra = np.linalg.qr(A)
    _, Rb = np.linalg.qr(B)
    return float(np.linalg.norm(Ra @ Rb.T))


def lowrank_norm(A, B):
    if A.shape[1] == 0:
        return 0.0
    _, Ra = np.linalg.qr(A)
    _, Rb = np.linalg.qr(B)
    return float(np.linalg.norm(Ra @ Rb.T))


def near_tags(octx):
    """(t, r) cluster ids of the oracle's near-threshold truncations
    (TruncCtx.near entries (idx, tag, k, s), tag = (kind, t_id, r_id))."""
    out = set()
    for e in octx.near:
        tag = e[1]
        if tag is not None and len(tag) >= 3:
            out.add((int(tag[1]), int(tag[2])))
    return sorted(out)


def near_block_set(d, octx):
    """Leaf blocks inside a near-threshold truncation's (t, r) block: the only
    blocks whose rank may differ (north star exemption)."""
    from oracle.summary import near_blocks
    return near_blocks(d, near_tags(octx))


def compare(dg, do, near_blocks=(), tol=1e-9, eps=0.0):
    """Per-block parity (north star): identical ranks except on near-flagged
    blocks (rank_mismatch must be a subset of near_blocks: see
    `unexplained_mismatch`); relative Frobenius difference <= tol on EVERY
    block whose rank agrees (the difference is measured rank-independently),
    and <= max(tol, 20 eps) on a near-flagged block whose rank flipped (one
    singular value at the threshold kept on one side, dropped on the other).
    Returns a report dict."""
    pg, po = leaf_payloads(dg), leaf_payloads(do)
    assert pg.keys() == po.keys()
    total = 0.0
    for b, v in po.items():
        total += np.linalg.norm(v[1]) ** 2 if v[0] == "dense" else lowrank_norm(v[1], v[2]) ** 2
    znorm = np.sqrt(total)
    rank_mis, worst, worst_b, worst_flip = [], 0.0, None, 0.0
    for b, vo in po.items():
        vg = pg[b]
        if vo[0] == "dense":
            den = max(np.linalg.norm(vo[1]), 1e-12 * znorm)
            rel = np.linalg.norm(vg[1] - vo[1]) / den
        else:
            if vg[1].shape[1] != vo[1].shape[1]:
                rank_mis.append(b)
            den = max(lowrank_norm(vo[1], vo[2]), 1e-12 * znorm)
            rel = lowrank_diff(vg[1], vg[2], vo[1], vo[2]) / den
        if vo[0] != "dense" and vg[1].shape[1] != vo[1].shape[1] and b in near_blocks:
            worst_flip = max(worst_flip, rel)
            continue
        if rel > worst:
            worst, worst_b = rel, b
    near_blocks = set(near_blocks)
    unexplained = [b for b in rank_mis if b not in near_blocks]
    if worst_flip > max(tol, 20.0 * eps):
        unexplained.append(("rank flip beyond the eps bound", worst_flip))
    return dict(rank_mismatch=rank_mis, unexplained_mismatch=unexplained,
                worst=worst, worst_block=worst_b, worst_flip=worst_flip, znorm=znorm)
