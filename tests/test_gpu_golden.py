"""Full-size GPU <-> oracle parity on BASELINE.json's configurations (pytest -m gpu).

Golden data come from `scripts/make_golden.py` (calls only oracle/; summary
format in oracle/summary.py): for EVERY leaf block of the oracle's result its
rank, exact Frobenius norm and a two-sided Gaussian sketch
Omega_L[t]^T Z_b Omega_R[r]; the built input's ranks and norms; the result
applied to two probe vectors; the (t, r) clusters of near-threshold
truncations.  The device side builds the same H-matrix with hm_build (trees
bit-identical, admissible blocks certified to 1e-12 against the exact SVD;
its ranks and per-block norms are checked against the oracle build first),
runs the operation in the launch configuration bench.py uses, exports the
result and summarises it with the same oracle/summary.py code.  Checks
(north star, BASELINE.json):
  * identical ranks on every block outside a near-threshold truncation's
    (t, r) block (mismatches must be a subset of the near-flagged blocks),
  * per-block difference estimate ||S_gpu - S_oracle||_F / k <= 1e-9 of
    max(||Z_b||_F, 1e-12 ||Z||_F) on every other block,
  * probes within 1e-9 relative.
"""
import json
import os

import numpy as np
import pytest

from hm_inputs import probe_vectors, sphere_points

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
TOL = 1e-9


@pytest.fixture(scope="module")
def hm():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1703_09085_b200 as hm
    return hm


@pytest.fixture(scope="module")
def ctx(hm):
    return hm.Context(0)


def _load(name):
    p = os.path.join(GOLD, name)
    if not os.path.exists(p):
        pytest.skip(f"golden file {name} not generated (scripts/make_golden.py)")
    g = np.load(p)
    return g, json.loads(str(g["meta"]))


def _check_build(G, g):
    """Device build vs the oracle build: ranks identical, norms <= 1e-9."""
    from oracle.summary import summarise_desc
    s = summarise_desc(G.export(), k=1)
    assert np.array_equal(s["ranks"], g["b_ranks"]), int(np.sum(s["ranks"] != g["b_ranks"]))
    znorm = np.sqrt(np.sum(g["b_fro"] ** 2))
    rel = np.abs(s["fro"] - g["b_fro"]) / np.maximum(g["b_fro"], 1e-12 * znorm)
    assert rel.max() <= TOL, rel.max()


def _check_result(out, g, meta):
    from oracle.summary import compare_summaries, near_blocks, summarise_desc
    d = out.export()
    k = g["sk"].shape[1]
    got = summarise_desc(d, k=k)
    ref = {key: g[key] for key in ("leaf_ids", "ranks", "fro", "sk")}
    allowed = near_blocks(d, [tuple(x) for x in g["near"]])
    rep = compare_summaries(got, ref, TOL, allowed, eps_bound=20 * meta["eps"])
    print(f"{meta['what']} cfg{meta['config']}: {rep['nleaves']} leaves, worst block diff {rep['worst']:.2e} "
          f"(block {rep['worst_block']}), near-flagged {len(allowed)}, rank mismatches {len(rep['rank_mismatch'])}")
    assert not rep["unexplained_mismatch"], rep["unexplained_mismatch"][:20]
    assert rep["worst"] <= TOL, rep
    assert rep["worst_allowed"] <= 20 * meta["eps"], rep
    return rep


def _probe(hm, M, n, perm, what):
    import torch
    v = probe_vectors(n, 2)[perm]
    xv = torch.from_numpy(v.T.copy()).cuda().T
    y = torch.zeros_like(xv)
    if what == "product":
        hm.matvec(M, xv, y)
    else:
        t = torch.zeros_like(xv)
        hm.matvec(M, xv, t, op=3 if what == "lr" else 5)   # R v | L^T v
        hm.matvec(M, t, y, op=2 if what == "lr" else 4)    # L (.)
    return y.cpu().numpy()


@pytest.mark.parametrize("cfg", [1, 4])
def test_product_golden(hm, ctx, cfg):
    g, meta = _load(f"product_cfg{cfg}.npz")
    x, w = sphere_points(meta["L"])
    G = ctx.build(x, w, meta["leaf"], 2.0, meta["eps"])
    _check_build(G, g)
    X, Y, Z = G.clone(), G.clone(), G.clone()
    hm.addmul(1.0, X, Y, Z, meta["eps"])
    st = ctx.last_stats()
    assert st["truncations"] == meta["truncations"]
    assert st["addproduct_calls"] == meta["addproduct"]
    _check_result(Z, g, meta)
    pr = _probe(hm, Z, len(w), G.perm, "product")
    assert np.linalg.norm(pr - g["probes"]) <= TOL * np.linalg.norm(g["probes"])


@pytest.mark.parametrize("kind,cfg", [("lr", 2), ("chol", 3), ("lr", 4), ("lr", 5)])
def test_factor_golden(hm, ctx, kind, cfg):
    """configs[1] (n=5120 H-LR), configs[2] (n=20480 H-Cholesky), the metric's
    n=81920 H-LR of configs[3]'s matrix and configs[4] (n=327680 H-LR)."""
    g, meta = _load(f"{kind}_cfg{cfg}.npz")
    x, w = sphere_points(meta["L"])
    G = ctx.build(x, w, meta["leaf"], 2.0, meta["eps"], kernel=0 if kind == "lr" else 1)
    _check_build(G, g)
    if kind == "lr":
        hm.lr(G, meta["eps"])
    else:
        hm.chol(G, meta["eps"], meta.get("shift", 0.0))
    st = ctx.last_stats()
    assert st["truncations"] == meta["truncations"]
    assert abs(st["min_pivot"] - meta["min_pivot"]) <= 1e-9 * meta["min_pivot"]
    _check_result(G, g, meta)
    pr = _probe(hm, G, len(w), G.perm, kind)
    assert np.linalg.norm(pr - g["probes"]) <= TOL * np.linalg.norm(g["probes"])


def _probe_residual_gpu(hm, G0, F, n, perm, kind):
    """||G v - L(R v)|| / ||G v|| (LR) or ||G v - L(L^T v)|| / ||G v|| with the
    device matvec on 8 probes."""
    import torch
    v = probe_vectors(n)[perm]
    x = torch.from_numpy(v.T.copy()).cuda().T
    gv = torch.zeros_like(x)
    hm.matvec(G0, x, gv)
    t = torch.zeros_like(x)
    y = torch.zeros_like(x)
    if kind == "lr":
        hm.matvec(F, x, t, op=3)      # R v
        hm.matvec(F, t, y, op=2)      # L (R v)
    else:
        hm.matvec(F, x, t, op=5)      # L^T v
        hm.matvec(F, t, y, op=4)      # L (L^T v)
    return float(torch.linalg.norm(gv - y) / torch.linalg.norm(gv))


@pytest.mark.parametrize("kind,L,leaf,eps", [
    ("lr", 4, 32, 1e-4),     # configs[1]
    ("chol", 5, 32, 1e-5),   # configs[2]
    ("lr", 6, 64, 1e-6),     # the metric's n = 81920 H-LR
])
def test_factor_probe_residual(hm, ctx, kind, L, leaf, eps):
    """Property valid at any size (north star check 4): probe residual of the
    device factors <= 50 eps (SURVEY #21), min pivot positive (no shift)."""
    x, w = sphere_points(L)
    G0 = ctx.build(x, w, leaf, 2.0, eps, kernel=0 if kind == "lr" else 1)
    F = G0.clone()
    (hm.lr if kind == "lr" else hm.chol)(F, eps)
    assert ctx.last_stats()["min_pivot"] > 0
    res = _probe_residual_gpu(hm, G0, F, len(w), G0.perm, kind)
    assert res <= 50 * eps, res
    print(f"{kind} n={len(w)} probe residual {res:.3e}")
