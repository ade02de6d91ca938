"""GPU <-> oracle parity of H-LR / H-Cholesky through the C-ABI (pytest -m gpu).

Both sides run the O8/O9 recursion with S2 accumulators on the same imported
H-matrix; per block: identical ranks and relative Frobenius difference <= 1e-9
of the in-place factors (north star)."""
import numpy as np
import pytest

from hm_inputs import probe_vectors, sphere_points
from oracle import kernel as K
from oracle.factor import chol as o_chol, lr as o_lr, probe_residual
from oracle.hmatrix import Problem, build, export, import_payload
from oracle.lowrank import TruncCtx
from tests.hm_compare import compare

pytestmark = pytest.mark.gpu
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


@pytest.mark.parametrize("L,leaf,eps", [(1, 4, 0.0), (2, 8, 0.0), (2, 8, 1e-4), (3, 32, 1e-4)])
@pytest.mark.parametrize("kind", ["lr", "chol"])
def test_factor_parity(hm, ctx, L, leaf, eps, kind):
    x, w = sphere_points(L)
    P = Problem(x, w, leaf, 2.0, kernel=K.KERNEL_SLP if kind == "lr" else K.KERNEL_SLP_SYM)
    G = build(P, eps)
    G0 = G.clone()
    octx = TruncCtx(eps)
    if kind == "lr":
        Fo, fo = o_lr(G.clone(), eps, ctx=octx)
    else:
        Fo, fo = o_chol(G.clone(), eps, ctx=octx)
    Gg = ctx.import_desc(export(G))
    (hm.lr if kind == "lr" else hm.chol)(Gg, eps)
    s = ctx.last_stats()
    assert s["truncations"] == octx.count
    dg = Gg.export()
    do = export(Fo)
    if kind == "chol":   # compare the lower triangle only (upper blocks are untouched inputs)
        for d in (dg, do):
            pass
    rep = compare(dg, do)
    assert not rep["rank_mismatch"] or octx.near, rep
    assert rep["worst"] <= TOL, rep
    v = probe_vectors(P.ct.n)[P.perm]
    Fg = import_payload(P.bt, dg)
    res = probe_residual(G0, Fg, v, kind)
    assert res <= max(50 * eps, 1e-12), res
    assert abs(s["min_pivot"] - fo.min_pivot) <= 1e-9 * fo.min_pivot


def test_chol_pivot_failure(hm, ctx):
    x, w = sphere_points(1)
    P = Problem(x, w, 4, 2.0, kernel=K.KERNEL_SLP_SYM)
    G = build(P, 1e-4)
    Gg = ctx.import_desc(export(G))
    with pytest.raises(hm.HMError) as ei:
        hm.chol(Gg, 1e-4, shift=-10.0)   # makes the matrix indefinite
    assert "EPIVOT" in str(ei.value) and "cluster" in str(ei.value)
