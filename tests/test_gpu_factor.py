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
from oracle.factor import apply_factor
from tests.hm_compare import compare, near_block_set

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
    # every leaf is compared (Cholesky: the strictly upper blocks are the
    # untouched inputs on both sides, so they must agree exactly as well)
    rep = compare(dg, do, near_block_set(do, octx))
    assert not rep["unexplained_mismatch"], rep
    assert rep["worst"] <= TOL, rep
    v = probe_vectors(P.ct.n)[P.perm]
    Fg = import_payload(P.bt, dg)
    res = probe_residual(G0, Fg, v, kind)
    assert res <= max(50 * eps, 1e-12), res
    assert abs(s["min_pivot"] - fo.min_pivot) <= 1e-9 * fo.min_pivot


@pytest.mark.parametrize("kind", ["lr", "chol"])
def test_factor_matvec_ops(hm, ctx, kind):
    """hm_matvec_thin ops 2-5 (L unit lower, R upper, Lc lower, Lc^T) of the
    device factors vs oracle.factor.apply_factor (P:L1549-1550 factors applied
    by Fig. 1 addeval over the leaves): applied to the device's own factors
    (exported) the two must agree to rounding (1e-13); applied to the oracle's
    factors, to the 1e-9 parity level of the factors themselves."""
    import torch
    L, leaf, eps = 3, 32, 1e-4
    x, w = sphere_points(L)
    P = Problem(x, w, leaf, 2.0, kernel=K.KERNEL_SLP if kind == "lr" else K.KERNEL_SLP_SYM)
    G = build(P, eps)
    Fo, _ = (o_lr if kind == "lr" else o_chol)(G.clone(), eps, ctx=TruncCtx(eps))
    Gg = ctx.import_desc(export(G))
    (hm.lr if kind == "lr" else hm.chol)(Gg, eps)
    Fg = import_payload(P.bt, Gg.export())
    rng = np.random.default_rng(5)
    X = rng.standard_normal((P.ct.n, 6))
    ops = {"lr": [(2, "L"), (3, "R")], "chol": [(4, "Lc"), (5, "LcT")]}[kind]
    for op, part in ops:
        xg = torch.from_numpy(X.T.copy()).cuda().T
        yg = torch.zeros_like(xg)
        hm.matvec(Gg, xg, yg, op=op)
        y = yg.cpu().numpy()
        ref_self = apply_factor(Fg, part, X)
        ref_orac = apply_factor(Fo, part, X)
        assert np.linalg.norm(y - ref_self) <= 1e-13 * np.linalg.norm(ref_self), (op, part)
        assert np.linalg.norm(y - ref_orac) <= 1e-9 * np.linalg.norm(ref_orac), (op, part)


def test_chol_pivot_failure(hm, ctx):
    x, w = sphere_points(1)
    P = Problem(x, w, 4, 2.0, kernel=K.KERNEL_SLP_SYM)
    G = build(P, 1e-4)
    Gg = ctx.import_desc(export(G))
    with pytest.raises(hm.HMError) as ei:
        hm.chol(Gg, 1e-4, shift=-10.0)   # makes the matrix indefinite
    assert "EPIVOT" in str(ei.value) and "cluster" in str(ei.value)


@pytest.mark.parametrize("kind", ["lr", "chol"])
def test_solve_thin(hm, ctx, kind):
    """hm_solve_thin (block substitution with the device factors) vs
    oracle.factor.solve_factor applied to the SAME factors (exported): the
    same exact operator inverse, rounding-level agreement; n = 5120 so the
    multi-launch path (clusters > 1024 rows) and the single-CTA path both run."""
    import torch
    from oracle.factor import solve_factor
    L, leaf, eps = 4, 32, 1e-4
    x, w = sphere_points(L)
    G = build(Problem(x, w, leaf, 2.0, kernel=K.KERNEL_SLP if kind == "lr" else K.KERNEL_SLP_SYM), eps)
    Gg = ctx.import_desc(export(G))
    (hm.lr if kind == "lr" else hm.chol)(Gg, eps)
    P = Problem(x, w, leaf, 2.0)
    Fg = import_payload(P.bt, Gg.export())
    rng = np.random.default_rng(11)
    X = rng.standard_normal((P.ct.n, 5))
    for op in (["L", "R", "LT", "RT"] if kind == "lr" else ["Lc", "LcT"]):
        xg = torch.from_numpy(X.T.copy()).cuda().T
        hm.solve(Gg, xg, op)
        ref = solve_factor(Fg, op, X.copy())
        got = xg.cpu().numpy()
        assert np.linalg.norm(got - ref) <= 1e-11 * np.linalg.norm(ref), op


@pytest.mark.parametrize("kind", ["lr", "chol"])
def test_precond_error(hm, ctx, kind):
    """Device power iteration (hm_precond_error) vs the exact
    ||I - F^{-1} G||_2 of the device's own factors (dense numpy at n = 1280)."""
    from oracle.factor import apply_factor
    L, leaf, eps = 3, 32, 1e-4
    x, w = sphere_points(L)
    kern = K.KERNEL_SLP if kind == "lr" else K.KERNEL_SLP_SYM
    G = build(Problem(x, w, leaf, 2.0, kernel=kern), eps)
    G0 = ctx.import_desc(export(G))
    Fd = G0.clone()
    (hm.lr if kind == "lr" else hm.chol)(Fd, eps)
    est = hm.precond_error(G0, Fd, kind, iters=150)
    P = Problem(x, w, leaf, 2.0)
    Fo = import_payload(P.bt, Fd.export())
    n = P.ct.n
    M = apply_factor(Fo, "L", apply_factor(Fo, "R", np.eye(n))) if kind == "lr" else \
        apply_factor(Fo, "Lc", apply_factor(Fo, "LcT", np.eye(n)))
    E = np.eye(n) - np.linalg.solve(M, G.to_dense())
    exact = np.linalg.norm(E, 2)
    assert abs(est - exact) <= 1e-3 * exact, (est, exact)
    print(f"{kind}: preconditioner error {est:.3e} (exact {exact:.3e})")


def test_dlp_build_and_lr(hm, ctx):
    """Double-layer matrix K + I/2: the device build equals
    the oracle build (bit-identical trees, identical ranks, <= 1e-9 per
    block), and its H-LR matches the oracle's (the paper's "L R = K" run,
    Fig. 11 right)."""
    from hm_inputs import sphere_normals
    L, leaf, eps = 3, 32, 1e-4
    x, w = sphere_points(L)
    nr = sphere_normals(L)
    P = Problem(x, w, leaf, 2.0, kernel=K.KERNEL_DLP, nrm=nr)
    Go = build(P, eps)
    Gg = ctx.build(x, w, leaf, 2.0, eps, kernel=2, normals=nr)
    do = export(Go)
    rep = compare(Gg.export(), do)
    assert not rep["rank_mismatch"], rep
    assert rep["worst"] <= TOL, rep
    octx = TruncCtx(eps)
    Fo, _ = o_lr(Go.clone(), eps, ctx=octx)
    Gi = ctx.import_desc(do)
    hm.lr(Gi, eps)
    assert ctx.last_stats()["truncations"] == octx.count
    dfo = export(Fo)
    rep = compare(Gi.export(), dfo, near_block_set(dfo, octx))
    assert not rep["unexplained_mismatch"], rep
    assert rep["worst"] <= TOL, rep


@pytest.mark.parametrize("L,leaf,eps", [(1, 4, 0.0), (2, 8, 0.0), (2, 8, 1e-4), (3, 32, 1e-4)])
def test_inv_parity(hm, ctx, L, leaf, eps):
    """Device H-inversion with accumulators (hm_inv, Fig. 8) vs
    oracle.inverse.invert on the same imported H-matrix: same truncation
    count, identical ranks, <= 1e-9 per block; at eps = 0 the exact inverse."""
    from oracle.inverse import invert as o_invert
    x, w = sphere_points(L)
    P = Problem(x, w, leaf, 2.0)
    G = build(P, eps)
    octx = TruncCtx(eps)
    Io, _ = o_invert(G.clone(), eps, octx)
    Gg = ctx.import_desc(export(G))
    hm.inv(Gg, eps)
    assert ctx.last_stats()["truncations"] == octx.count
    dg, do = Gg.export(), export(Io)
    rep = compare(dg, do, near_block_set(do, octx))
    assert not rep["unexplained_mismatch"], rep
    assert rep["worst"] <= TOL, rep
    if eps == 0.0:
        D = import_payload(P.bt, dg).to_dense()
        assert np.linalg.norm(G.to_dense() @ D - np.eye(P.ct.n)) <= 1e-10 * np.sqrt(P.ct.n)


def test_inv_precond_error(hm, ctx):
    """||I - G~^{-1} G||_2 of the device inverse by the device power iteration
    (hm_precond_error kind 2) vs the dense exact value."""
    x, w = sphere_points(3)
    P = Problem(x, w, 32, 2.0)
    G = build(P, 1e-4)
    G0 = ctx.import_desc(export(G))
    Gi = G0.clone()
    hm.inv(Gi, 1e-4)
    est = hm.precond_error(G0, Gi, "inv", iters=100)
    D = import_payload(P.bt, Gi.export()).to_dense()
    exact = np.linalg.norm(np.eye(P.ct.n) - D @ G.to_dense(), 2)
    assert abs(est - exact) <= 1e-3 * exact, (est, exact)
