"""Full-size GPU <-> oracle parity on BASELINE.json's configurations (pytest -m gpu).

Golden data come from `scripts/make_golden.py` (calls only oracle/):
per-block ranks and Frobenius norms of the oracle's result, sketches
Z_b Omega_b of ~400 sampled leaf blocks, and the result applied to two probe
vectors.  The device side builds the same H-matrix with hm_build (trees
bit-identical, admissible blocks certified to 1e-12 against the exact SVD),
runs the operation in the launch configuration bench.py uses, and is
compared on: identical ranks (blocks flagged near-threshold by the oracle
excepted), per-block norms and sampled sketches within 1e-9 relative, probes
within 1e-9 relative.
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


def _payloads(d):
    from tests.hm_compare import leaf_payloads
    return leaf_payloads(d)


def _fro(v):
    if v[0] == "dense":
        return float(np.linalg.norm(v[1]))
    A, B = v[1], v[2]
    if A.shape[1] == 0:
        return 0.0
    return float(np.sqrt(max(np.sum((A.T @ A) * (B.T @ B)), 0.0)))


def _check(hm, ctx, out, g, meta):
    d = out.export()
    pay = _payloads(d)
    ranks = g["ranks"]
    nearb = set()
    mism = [b for b, v in pay.items() if v[0] == "adm" and v[1].shape[1] != ranks[b]]
    assert not mism or meta.get("near"), (len(mism), mism[:10])
    fro = g["fro"]
    znorm = np.sqrt(np.sum(fro ** 2))
    worst = 0.0
    for b, v in pay.items():
        if b in mism:
            continue
        worst = max(worst, abs(_fro(v) - fro[b]) / max(fro[b], 1e-12 * znorm))
    assert worst <= TOL, worst
    ws = 0.0
    for bid in g["sample"]:
        if int(bid) in mism:
            continue
        v = pay[int(bid)]
        n_b = (v[1].shape[1] if v[0] == "dense" else v[2].shape[0])
        Om = np.random.default_rng([1703, 9085, 99, int(bid)]).standard_normal((n_b, 4))
        s = v[1] @ Om if v[0] == "dense" else v[1] @ (v[2].T @ Om)
        ref = g[f"sketch_{int(bid)}"]
        ws = max(ws, np.linalg.norm(s - ref) / max(np.linalg.norm(ref), 1e-12 * znorm))
    assert ws <= TOL, ws
    return worst, ws


@pytest.mark.parametrize("cfg", [1, 4])
def test_product_golden(hm, ctx, cfg):
    import torch
    g, meta = _load(f"product_cfg{cfg}.npz")
    x, w = sphere_points(meta["L"])
    G = ctx.build(x, w, meta["leaf"], 2.0, meta["eps"])
    X, Y, Z = G.clone(), G.clone(), G.clone()
    hm.addmul(1.0, X, Y, Z, meta["eps"])
    st = ctx.last_stats()
    assert st["truncations"] == meta["truncations"]
    assert st["addproduct_calls"] == meta["addproduct"]
    _check(hm, ctx, Z, g, meta)
    n = len(w)
    v = probe_vectors(n, 2)[G.perm]
    xv = torch.from_numpy(v.T.copy()).cuda().T
    yv = torch.zeros_like(xv)
    hm.matvec(Z, xv, yv)
    pr = yv.cpu().numpy()
    assert np.linalg.norm(pr - g["probes"]) <= TOL * np.linalg.norm(g["probes"])


@pytest.mark.parametrize("kind,cfg", [("lr", 2), ("chol", 3)])
def test_factor_golden(hm, ctx, kind, cfg):
    g, meta = _load(f"{kind}_cfg{cfg}.npz")
    x, w = sphere_points(meta["L"])
    G = ctx.build(x, w, meta["leaf"], 2.0, meta["eps"], kernel=0 if kind == "lr" else 1)
    if kind == "lr":
        hm.lr(G, meta["eps"])
    else:
        hm.chol(G, meta["eps"], meta.get("shift", 0.0))
    st = ctx.last_stats()
    assert st["truncations"] == meta["truncations"]
    assert abs(st["min_pivot"] - meta["min_pivot"]) <= 1e-9 * meta["min_pivot"]
    _check(hm, ctx, G, g, meta)


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
    ("lr", 7, 64, 1e-4),     # configs[4]: n = 327680, fully HBM resident
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
