"""GPU <-> oracle parity through the C-ABI (pytest -m gpu).

The oracle (oracle/, CPU, FP64) builds the H-matrix; the same host
description is imported into libhm; both sides run Z <- Z + alpha X Y with
the S2 schedule; per admissible block the ranks must be identical and the
relative Frobenius difference <= 1e-9 (north star; BASELINE.json), dense
blocks entrywise in relative Frobenius.
"""
import numpy as np
import pytest

from hm_inputs import random_points, sphere_points
from oracle.hmatrix import Problem, build, export, matvec as o_matvec
from oracle.lowrank import TruncCtx, trunc
from oracle.product import addmul_s2
from tests.hm_compare import compare, leaf_payloads, lowrank_diff, lowrank_norm, near_block_set

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


def _prescribed(rng, m, n, s, junk):
    q = len(s)
    U, _ = np.linalg.qr(rng.standard_normal((m, q)))
    V, _ = np.linalg.qr(rng.standard_normal((n, q)))
    As, Bs = [U * s], [V]
    for _ in range(junk):
        X = rng.standard_normal((m, 2))
        Y = rng.standard_normal((n, 2))
        As += [X, -X]
        Bs += [Y, Y]
    return np.hstack(As), np.hstack(Bs)


def _assert_one_orthonormal(U, V, k):
    """The device TRUNC returns one orthonormal factor (the short side of the
    SVD'd matrix, reading R7c); the other carries the singular values."""
    eu = np.abs(U.T @ U - np.eye(k)).max() if k else 0.0
    ev = np.abs(V.T @ V - np.eye(k)).max() if k else 0.0
    assert min(eu, ev) <= 1e-12, (eu, ev)


@pytest.mark.parametrize("eps", [1e-4, 1e-6])
def test_trunc_kernel_prescribed_sigma(hm, ctx, eps):
    """Batched TRUNC vs the closed-form Eckart-Young rank/error
    and vs the oracle's TRUNC on the same stacks; sizes span every path
    (QR both sides, one side, dense; smem buckets and the global path)."""
    rng = np.random.default_rng(12)
    shapes = [(40, 30, 12, 0), (200, 150, 20, 2), (64, 64, 64, 1), (300, 40, 25, 3), (17, 500, 16, 2),
              (130, 170, 90, 4), (5, 3, 3, 0), (1, 1, 1, 0), (700, 650, 60, 3), (260, 240, 240, 2)]
    stacks, svals = [], []
    for m, n, q, junk in shapes:
        s = 10.0 ** (-0.31 * np.arange(q))    # no singular value sits on the eps threshold
        A, B = _prescribed(rng, m, n, s, junk)
        stacks.append((A, B))
        svals.append(s)
    out, ranks, sig = hm.test_trunc_batched(ctx, stacks, eps)
    for (A, B), (U, V), k, s in zip(stacks, out, ranks, svals):
        tot = np.sum(s ** 2)
        kk = next(j for j in range(len(s) + 1) if np.sum(s[j:] ** 2) <= eps ** 2 * tot)
        assert k == kk
        err = np.linalg.norm(A @ B.T - U @ V.T)
        np.testing.assert_allclose(err, np.sqrt(np.sum(s[k:] ** 2)), rtol=1e-7, atol=1e-13 * np.linalg.norm(A) * np.linalg.norm(B))
        _assert_one_orthonormal(U, V, k)
        Uo, Vo = trunc(A, B, TruncCtx(eps))
        assert Uo.shape[1] == k
        assert lowrank_diff(U, V, Uo, Vo) <= TOL * lowrank_norm(Uo, Vo) + 1e-14


def test_trunc_kernel_tall(hm, ctx):
    """Tall stacks taking the TSQR route (factor rows > 1536: chunked QR, stacked
    R's, up to five levels, ragged last chunks) -- same closed-form checks."""
    eps = 1e-6
    rng = np.random.default_rng(21)
    shapes = [(5000, 3000, 40, 2), (40000, 200, 150, 1), (1700, 1600, 376, 1), (2000, 30, 10, 0),
              (60000, 400, 300, 2), (3100, 2900, 500, 0)]
    stacks, svals = [], []
    for m, n, q, junk in shapes:
        s = 10.0 ** (-0.13 * np.arange(q))
        A, B = _prescribed(rng, m, n, s, junk)
        stacks.append((A, B))
        svals.append(s)
    out, ranks, _ = hm.test_trunc_batched(ctx, stacks, eps)
    for (A, B), (U, V), k, s in zip(stacks, out, ranks, svals):
        kk = next(j for j in range(len(s) + 1) if np.sum(s[j:] ** 2) <= eps ** 2 * np.sum(s ** 2))
        assert k == kk
        # ||A B^T - U V^T||_F = ||R1 R2^T|| with [A, -U] = Q1 R1, [B, V] = Q2 R2
        R1 = np.linalg.qr(np.hstack([A, -U]), mode="r")
        R2 = np.linalg.qr(np.hstack([B, V]), mode="r")
        err = np.linalg.norm(R1 @ R2.T)
        tail = np.sqrt(np.sum(s[k:] ** 2))
        scale = np.linalg.norm(A) * np.linalg.norm(B)   # rounding level of the stack itself
        assert abs(err - tail) <= 1e-6 * tail + 1e-13 * scale, (err, tail, scale)
        _assert_one_orthonormal(U, V, k)


def test_trunc_kernel_stepped_qr(hm, ctx):
    """Batches large enough (>= 32 QR jobs per shared-memory bucket) to take
    the stepped QR (k_qrs_panel + k_qrs_update, qr.cu): ragged column counts
    (not multiples of 16), every bucket (<= 384 / 768 / 1536 rows), jobs that
    run out of columns at different panel steps -- closed form + oracle TRUNC."""
    eps = 1e-6
    rng = np.random.default_rng(77)
    shapes = []
    for i in range(40):
        m = 200 + (i * 7) % 180
        shapes.append((m, m - 11, 10 + i % 25, i % 4))
        m = 500 + (i * 13) % 260
        shapes.append((m, m - 30, 20 + (i * 3) % 70, i % 3))
        m = 900 + (i * 29) % 600
        shapes.append((m, 800 + (i * 17) % 500, 30 + (i * 5) % 120, i % 5))
    stacks, svals = [], []
    for m, n, q, junk in shapes:
        s = 10.0 ** (-0.17 * np.arange(q))
        A, B = _prescribed(rng, m, n, s, junk)
        stacks.append((A, B))
        svals.append(s)
    out, ranks, _ = hm.test_trunc_batched(ctx, stacks, eps)
    for (A, B), (U, V), k, s in zip(stacks, out, ranks, svals):
        kk = next(j for j in range(len(s) + 1) if np.sum(s[j:] ** 2) <= eps ** 2 * np.sum(s ** 2))
        assert k == kk
        _assert_one_orthonormal(U, V, k)
        Uo, Vo = trunc(A, B, TruncCtx(eps))
        assert Uo.shape[1] == k
        assert lowrank_diff(U, V, Uo, Vo) <= TOL * lowrank_norm(Uo, Vo) + 1e-14


def test_trunc_kernel_reg_qr(hm, ctx):
    """Stacks whose QR jobs cover the five row classes of the register-panel
    QR (qr_reg.cu: <= 128 / 256 / 384 / 512 / 768 rows), ragged column counts
    (last panel < 16 columns, l = 17 .. 133), few and many jobs, TSQR chunk
    stacks (2 l .. 5 l rows) and pre-QR of M -- closed form + oracle TRUNC."""
    eps = 1e-6
    rng = np.random.default_rng(2718)
    shapes = []
    for i in range(12):
        shapes.append((130 + 19 * i, 125 + 17 * i, 17 + 9 * i, i % 3))        # classes 1-2, both sides QR'd
        shapes.append((400 + 30 * i, 90 + 5 * i, 33 + 8 * i, i % 2))          # classes 3-4 one-sided
        shapes.append((1600 + 400 * i, 300 + 20 * i, 20 + 6 * i, 1))          # TSQR: chunk stacks of 2-7 l rows
    shapes += [(768, 767, 133, 0), (385, 384, 100, 1), (257, 256, 31, 2), (129, 128, 47, 0), (513, 512, 64, 1)]
    # M = R_A R_B^T of 112 .. 167 columns: the SVD's spill mode (svd.cu), then the global workspace
    shapes += [(300, 290, 113, 0), (320, 310, 150, 1), (500, 450, 160, 0), (400, 380, 167, 0), (420, 400, 166, 1)]
    stacks, svals = [], []
    for m, n, q, junk in shapes:
        s = 10.0 ** (-0.21 * np.arange(q))
        A, B = _prescribed(rng, m, n, s, junk)
        stacks.append((A, B))
        svals.append(s)
    for batch in (stacks, stacks[:3]):
        out, ranks, _ = hm.test_trunc_batched(ctx, batch, eps)
        for (A, B), (U, V), k, s in zip(batch, out, ranks, svals):
            kk = next(j for j in range(len(s) + 1) if np.sum(s[j:] ** 2) <= eps ** 2 * np.sum(s ** 2))
            assert k == kk
            _assert_one_orthonormal(U, V, k)
            Uo, Vo = trunc(A, B, TruncCtx(eps))
            assert Uo.shape[1] == k
            assert lowrank_diff(U, V, Uo, Vo) <= TOL * lowrank_norm(Uo, Vo) + 1e-14


def test_trunc_kernel_degenerate(hm, ctx):
    rng = np.random.default_rng(3)
    R = (rng.standard_normal((30, 4)), rng.standard_normal((25, 4)))
    stacks = [(np.hstack([R[0], -R[0]]), np.hstack([R[1], R[1]])),        # exact cancellation
              (np.zeros((12, 3)), np.zeros((9, 3))),                         # zero
              (rng.standard_normal((8, 0)), rng.standard_normal((6, 0)))]    # empty stack
    out, ranks, _ = hm.test_trunc_batched(ctx, stacks, 1e-8)
    assert ranks[1] == 0 and ranks[2] == 0
    U, V = out[0]
    assert ranks[0] == 0 or np.linalg.norm(U @ V.T) <= 1e-12 * np.linalg.norm(R[0] @ R[1].T)


def _cfg(L, leaf, eps):
    x, w = sphere_points(L)
    P = Problem(x, w, leaf, 2.0)
    G = build(P, eps)
    return P, G


@pytest.mark.parametrize("L,leaf,eps,alpha", [
    (1, 4, 0.0, 1.0),       # n=80: Fig. 5 / Fig. 7 branches, exact arithmetic
    (2, 8, 0.0, -0.5),      # n=320: + nested virtual recursion, eps = 0
    (2, 8, 1e-4, 1.0),      # n=320, eps = 1e-4
    (3, 32, 1e-4, 1.0),     # config 1 (BASELINE.json configs[0])
])
def test_addmul_parity(hm, ctx, L, leaf, eps, alpha):
    P, G = _cfg(L, leaf, eps)
    octx = TruncCtx(eps)
    Zo, octx, st = addmul_s2(alpha, G.clone(), G.clone(), G.clone(), eps, ctx=octx)
    do = export(Zo)
    Gg = ctx.import_desc(export(G))
    X, Y, Z = Gg.clone(), Gg.clone(), Gg.clone()
    hm.addmul(alpha, X, Y, Z, eps)
    dg = Z.export()
    s = ctx.last_stats()
    assert s["addproduct_calls"] == st.addproduct
    assert s["truncations"] == octx.count
    rep = compare(dg, do, near_block_set(do, octx))
    assert not rep["unexplained_mismatch"], rep
    assert rep["worst"] <= TOL, rep
    if eps == 0.0:
        Gd = G.to_dense()
        ref = Gd + alpha * Gd @ Gd
        from oracle.hmatrix import import_payload
        Zg = import_payload(P.bt, dg).to_dense()
        assert np.linalg.norm(Zg - ref) <= 1e-12 * np.linalg.norm(ref)


def test_addmul_and_lr_bit_reproducible(hm, ctx, monkeypatch):
    """No atomics, disjoint outputs per CTA (the lock-free update claim,
    P:L1333-1336): repeated runs of the product (the level built by several
    host threads: n = 5120 has levels above the 20 000-term threshold) and of
    the H-LR give bit-identical ranks, factors and dense leaves."""
    from hm_inputs import sphere_points
    x, w = sphere_points(4)
    G = ctx.build(x, w, 32, 2.0, 1e-4)
    outs = []
    for _ in range(2):
        X, Y, Z = G.clone(), G.clone(), G.clone()
        hm.addmul(1.0, X, Y, Z, 1e-4)
        outs.append(Z.export())
        for M in (X, Y, Z):
            M.free()
    assert np.array_equal(outs[0]["bl_rank"], outs[1]["bl_rank"])
    assert np.array_equal(outs[0]["factors"], outs[1]["factors"])
    assert np.array_equal(outs[0]["dense"], outs[1]["dense"])
    outs = []
    for _ in range(2):
        F = G.clone()
        hm.lr(F, 1e-4)
        outs.append(F.export())
        F.free()
    assert np.array_equal(outs[0]["bl_rank"], outs[1]["bl_rank"])
    assert np.array_equal(outs[0]["factors"], outs[1]["factors"])
    assert np.array_equal(outs[0]["dense"], outs[1]["dense"])


def test_addmul_distinct_operands(hm, ctx):
    """X != Y != Z (ragged random geometry, odd n)."""
    x, w = random_points(333, 4)
    P = Problem(x, w, 7, 2.0)
    X = build(P, 1e-6)
    Y = X.clone()
    for k in Y.A:
        Y.B[k] = 0.5 * Y.B[k]
    for k in Y.N:
        Y.N[k] = Y.N[k].T.copy() if Y.N[k].shape[0] == Y.N[k].shape[1] else Y.N[k] * 2.0
    Z = X.clone()
    Zo, octx, _ = addmul_s2(0.7, X.clone(), Y.clone(), Z.clone(), 1e-6)
    Xg, Yg, Zg = ctx.import_desc(export(X)), ctx.import_desc(export(Y)), ctx.import_desc(export(Z))
    hm.addmul(0.7, Xg, Yg, Zg, 1e-6)
    do = export(Zo)
    rep = compare(Zg.export(), do, near_block_set(do, octx))
    assert not rep["unexplained_mismatch"], rep
    assert rep["worst"] <= TOL, rep


def test_addmul_rejects_alias(hm, ctx):
    P, G = _cfg(1, 4, 1e-4)
    Gg = ctx.import_desc(export(G))
    with pytest.raises(hm.HMError) as ei:
        hm.addmul(1.0, Gg, Gg, Gg, 1e-4)
    assert "ESTRUCT" in str(ei.value)


@pytest.mark.parametrize("L,leaf,kernel", [(3, 32, 0), (2, 8, 1)])
def test_build_parity(hm, ctx, L, leaf, kernel):
    """hm_build on the device vs the oracle build: identical trees (bit-exact
    integer arrays and bounding boxes), identical ranks, per-block <= 1e-9."""
    x, w = sphere_points(L)
    eps = 1e-4
    P = Problem(x, w, leaf, 2.0, kernel=kernel)
    Go = build(P, eps)
    do = export(Go)
    Gg = ctx.build(x, w, leaf, 2.0, eps, kernel=kernel)
    dg = Gg.export()
    for k in ("cl_start", "cl_size", "cl_son0", "cl_nsons", "cl_level", "bl_row", "bl_col", "bl_kind",
              "bl_son0", "bl_nsons"):
        np.testing.assert_array_equal(dg[k], do[k], err_msg=k)
    np.testing.assert_array_equal(dg["perm"], do["perm"])
    np.testing.assert_array_equal(dg["cl_bbox"], do["cl_bbox"])
    rep = compare(dg, do)
    assert not rep["rank_mismatch"], rep
    assert rep["worst"] <= TOL, rep


def test_matvec(hm, ctx):
    import torch
    P, G = _cfg(2, 8, 1e-4)
    Gg = ctx.import_desc(export(G))
    n = P.ct.n
    rng = np.random.default_rng(0)
    X = rng.standard_normal((n, 8))
    Y0 = rng.standard_normal((n, 8))
    for op in (0, 1):
        ref = Y0 * 0.5
        o_matvec(G, 2.0, X, ref, trans=bool(op))
        xg = torch.from_numpy(X.T.copy()).cuda().T
        yg = torch.from_numpy(Y0.T.copy()).cuda().T
        hm.matvec(Gg, xg, yg, alpha=2.0, beta=0.5, op=op)
        np.testing.assert_allclose(yg.cpu().numpy(), ref, atol=1e-13 * np.abs(ref).max())


def test_eval_batched_kernel(hm, ctx):
    """hm_test_eval_batched (Fig. 1 addeval / addevaltrans) vs the
    oracle's recursive addeval / addevaltrans on the same H-matrix, for blocks
    of every kind (subdivided, admissible, dense), both orientations, ragged
    widths, with and without the row-group split of large jobs: the sums run
    over the same leaves, so the results agree to rounding (1e-13)."""
    from oracle.hmatrix import addeval, addevaltrans
    x, w = random_points(700, 9)
    P = Problem(x, w, 16, 2.0)
    G = build(P, 1e-6)
    Gg = ctx.import_desc(export(G))
    rng = np.random.default_rng(4)
    blocks = [P.bt.root] + [b for b in P.bt.blocks if b.kind == 0][1:6] + \
        [b for b in P.bt.blocks if b.kind == 1][:4] + [b for b in P.bt.blocks if b.kind == 2][:4]
    jobs, refs = [], []
    for i, b in enumerate(blocks):
        for trans in (0, 1):
            wdt = int(rng.integers(1, 40))
            coef = float(rng.uniform(-2, 2))
            rows_in = b.t.size if trans else b.s.size
            V = rng.standard_normal((rows_in, wdt))
            ref = np.zeros((b.s.size if trans else b.t.size, wdt))
            (addevaltrans if trans else addeval)(G, b, coef, V, ref)
            jobs.append((b.id, trans, coef, V))
            refs.append(ref)
    for thr in (0.0, 1e3):   # production rule / force the row-group split
        outs = hm.test_eval_batched(Gg, jobs, split_threshold=thr)
        for (bid, trans, _, _), o, ref in zip(jobs, outs, refs):
            assert np.linalg.norm(o - ref) <= 1e-13 * max(np.linalg.norm(ref), 1e-300), (bid, trans, thr)


@pytest.mark.parametrize("presum", ["1", "0"])
def test_addmul_identity_presum_parity(hm, ctx, presum, monkeypatch):
    """Identity pre-summing (reading R7d) on / off: same truncation count, the
    same ranks and <= 1e-9 per-block agreement with the oracle either way
    (the truncated exact matrices are identical)."""
    monkeypatch.setenv("HM_NO_PRESUM", "0" if presum == "1" else "1")
    P, G = _cfg(3, 16, 1e-6)
    octx = TruncCtx(1e-6)
    Zo, octx, _ = addmul_s2(1.0, G.clone(), G.clone(), G.clone(), 1e-6, ctx=octx)
    do = export(Zo)
    Gg = ctx.import_desc(export(G))
    X, Y, Z = Gg.clone(), Gg.clone(), Gg.clone()
    hm.addmul(1.0, X, Y, Z, 1e-6)
    assert ctx.last_stats()["truncations"] == octx.count
    rep = compare(Z.export(), do, near_block_set(do, octx))
    assert not rep["unexplained_mismatch"], rep
    assert rep["worst"] <= TOL, rep
    print(f"presum={presum}: trunc_cols {ctx.last_stats()['trunc_cols']} (oracle printed-branch {octx.cols})")


def test_flush_capture_replay(hm, ctx):
    """Standalone batched flush (BASELINE configs[3] timing mode):
    every captured level's TRUNC batch replayed from its captured stacks
    reproduces the in-situ ranks (same inputs, same kernels)."""
    P, G = _cfg(3, 32, 1e-4)
    Gg = ctx.import_desc(export(G))
    X, Y, Z = Gg.clone(), Gg.clone(), Gg.clone()
    hm.flush_capture(ctx, (1 << 63) - 1)
    hm.addmul(1.0, X, Y, Z, 1e-4)
    info = hm.flush_capture_info(ctx)
    assert len(info) >= 3
    ntr = 0
    for lev, L in enumerate(info):
        assert L["has_data"]
        ms, rs = hm.flush_replay(ctx, lev, 1e-4, reps=2)
        assert rs == int(L["k"].sum()), (lev, rs, int(L["k"].sum()))
        assert ms > 0
        ntr += len(L["m"])
    # level batches hold every truncation except the rkmerge ones (T4)
    assert 0 < ntr <= ctx.last_stats()["truncations"]
    hm.flush_capture_free(ctx)


@pytest.mark.parametrize("L,leaf,eps,alpha", [
    (1, 4, 0.0, 1.0),       # n=80: exact arithmetic, every S0 branch incl. temporaries
    (2, 8, 1e-4, -0.5),     # n=320: nested temporaries + rkmerge
    (3, 32, 1e-4, 1.0),     # config 1
])
def test_addmul_std_parity(hm, ctx, L, leaf, eps, alpha):
    """Device standard product S0 (hm_addmul_std) vs oracle.product.addmul_s0
    (P:L806-883): same truncation count, identical ranks, <= 1e-9 per block;
    at eps = 0 the exact product."""
    from oracle.product import addmul_s0
    P, G = _cfg(L, leaf, eps)
    octx = TruncCtx(eps)
    Zo, octx, st = addmul_s0(alpha, G.clone(), G.clone(), G.clone(), eps, ctx=octx)
    do = export(Zo)
    Gg = ctx.import_desc(export(G))
    X, Y, Z = Gg.clone(), Gg.clone(), Gg.clone()
    hm.addmul_std(alpha, X, Y, Z, eps)
    s = ctx.last_stats()
    assert s["addproduct_calls"] == st.addproduct
    assert s["truncations"] == octx.count
    dg = Z.export()
    rep = compare(dg, do, near_block_set(do, octx))
    assert not rep["unexplained_mismatch"], rep
    assert rep["worst"] <= TOL, rep
    if eps == 0.0:
        Gd = G.to_dense()
        ref = Gd + alpha * Gd @ Gd
        from oracle.hmatrix import import_payload
        Zg = import_payload(P.bt, dg).to_dense()
        assert np.linalg.norm(Zg - ref) <= 1e-12 * np.linalg.norm(ref)
    print(f"S0 n={P.ct.n}: {s['truncations']} truncations in {s['levels']} rounds")


def test_addmul_std_vs_accumulated(hm, ctx):
    """The paper's claim in numbers (Fig. 9): on the same input
    the standard product truncates far more often than the accumulated one,
    and both stay within the eps bound of each other (north-star check 3)."""
    P, G = _cfg(3, 32, 1e-4)
    Gg = ctx.import_desc(export(G))
    Z2 = Gg.clone()
    hm.addmul(1.0, Gg.clone(), Gg.clone(), Z2, 1e-4)
    t2 = ctx.last_stats()["truncations"]
    Z0 = Gg.clone()
    hm.addmul_std(1.0, Gg.clone(), Gg.clone(), Z0, 1e-4)
    t0 = ctx.last_stats()["truncations"]
    assert t0 > 3 * t2, (t0, t2)
    from oracle.hmatrix import import_payload
    A = import_payload(P.bt, Z2.export()).to_dense()
    B = import_payload(P.bt, Z0.export()).to_dense()
    depth = P.bt.depth()
    assert np.linalg.norm(A - B) <= 2 * (depth + 2) * 1e-4 * np.linalg.norm(A)


def test_torch_allocator_hook(hm):
    """hm_allocator hook (include/hm.h) with torch's caching allocator: the
    library's pools come from torch (torch.cuda.memory_allocated grows while
    matrices live, returns after the context is destroyed) and the product is
    unchanged (same result as with the private pool)."""
    import torch
    P, G = _cfg(2, 8, 1e-4)
    d = export(G)
    c1 = hm.Context(0)
    X, Y, Z = c1.import_desc(d), c1.import_desc(d), c1.import_desc(d)
    hm.addmul(1.0, X, Y, Z, 1e-4)
    ref = Z.export()
    c1.close()
    base = torch.cuda.memory_allocated()
    c2 = hm.Context(0, torch_allocator=True)
    X, Y, Z = c2.import_desc(d), c2.import_desc(d), c2.import_desc(d)
    assert torch.cuda.memory_allocated() > base
    hm.addmul(1.0, X, Y, Z, 1e-4)
    rep = compare(Z.export(), ref)
    assert not rep["rank_mismatch"] and rep["worst"] <= 1e-12, rep
    c2.close()
    torch.cuda.synchronize()
    assert torch.cuda.memory_allocated() == base
