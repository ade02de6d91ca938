"""Pins for the H-matrix container, build, addeval/addevaltrans, rkupdate.

  * addeval / addevaltrans are exact (Fig. 1): equal the dense
    product of the assembled matrix to 1e-13.
  * build at eps = 0 reproduces the dense kernel matrix (leaves tile I x I).
  * build at eps > 0: per admissible block the error equals the closed-form
    Eckart-Young tail of that block's singular values.
  * the certified randomized compression equals the exact truncated SVD
    where both run.
  * rkupdate at eps = 0 is exact (Fig. 3).
"""
import numpy as np
import pytest

from hm_inputs import random_points, sphere_points
from oracle.hmatrix import (Problem, _randomized_trunc, addeval, addevaltrans, build, export,
                            import_payload, rkupdate)
from oracle.lowrank import TruncCtx, choose_rank
from oracle.trees import ADM, DENSE


@pytest.fixture(scope="module")
def small():
    x, w = sphere_points(2)
    P = Problem(x, w, 8, 2.0)
    return P, build(P, 1e-4), P.dense()


def test_build_eps0_is_dense():
    x, w = random_points(150, 3)
    P = Problem(x, w, 10, 2.0)
    H = build(P, 0.0)
    D = P.dense()
    np.testing.assert_allclose(H.to_dense(), D, rtol=0, atol=1e-13 * np.abs(D).max())


def test_build_block_errors_eckart_young(small):
    P, H, D = small
    for b in P.bt.leaves():
        Gb = D[b.t.start:b.t.start + b.t.size, b.s.start:b.s.start + b.s.size]
        if b.kind == DENSE:
            np.testing.assert_array_equal(H.N[b.id], Gb)
            continue
        s = np.linalg.svd(Gb, compute_uv=False)
        err = np.linalg.norm(Gb - H.A[b.id] @ H.B[b.id].T)
        k = H.rank(b)
        np.testing.assert_allclose(err, np.sqrt(np.sum(s[k:] ** 2)), rtol=1e-6, atol=1e-13 * s[0])
        assert np.sum(s[k:] ** 2) <= 1e-8 * np.sum(s ** 2) * (1 + 1e-12)
        if k > 0:
            assert np.sum(s[k - 1:] ** 2) > 1e-8 * np.sum(s ** 2) * (1 - 1e-12)


def test_randomized_equals_exact(small):
    P, H, D = small
    big = max((b for b in P.bt.leaves() if b.kind == ADM), key=lambda b: b.t.size * b.s.size)
    Gb = D[big.t.start:big.t.start + big.t.size, big.s.start:big.s.start + big.s.size]
    A, B, res = _randomized_trunc(Gb, 1e-4, 0)
    assert res <= 1e-12
    assert A.shape[1] == H.rank(big)
    np.testing.assert_allclose(A @ B.T, H.A[big.id] @ H.B[big.id].T, atol=1e-11 * np.linalg.norm(Gb))


@pytest.mark.parametrize("c", [1, 5])
def test_addeval_exact(small, c):
    P, H, D = small
    Hd = H.to_dense()
    rng = np.random.default_rng(c)
    for b in [P.bt.root] + P.bt.blocks[1:40:7]:
        sub = Hd[b.t.start:b.t.start + b.t.size, b.s.start:b.s.start + b.s.size]
        X = rng.standard_normal((b.s.size, c))
        Y = rng.standard_normal((b.t.size, c))
        Y0 = Y.copy()
        addeval(H, b, -0.7, X, Y)
        np.testing.assert_allclose(Y, Y0 - 0.7 * sub @ X, atol=1e-13 * (1 + np.abs(Y0).max()))
        X0 = X.copy()
        Yt = rng.standard_normal((b.t.size, c))
        addevaltrans(H, b, 1.3, Yt, X)
        np.testing.assert_allclose(X, X0 + 1.3 * sub.T @ Yt, atol=1e-13 * (1 + np.abs(X0).max()))


def test_rkupdate_exact_eps0(small):
    P, H, D = small
    H2 = H.clone()
    Hd = H.to_dense()
    rng = np.random.default_rng(9)
    b = P.bt.blocks[1]
    A = rng.standard_normal((b.t.size, 3))
    B = rng.standard_normal((b.s.size, 3))
    rkupdate(H2, b, 0.5, A, B, TruncCtx(0.0))
    ref = Hd.copy()
    ref[b.t.start:b.t.start + b.t.size, b.s.start:b.s.start + b.s.size] += 0.5 * A @ B.T
    np.testing.assert_allclose(H2.to_dense(), ref, atol=1e-12 * np.abs(ref).max())


def test_export_import_roundtrip(small):
    P, H, D = small
    d = export(H)
    H2 = import_payload(P.bt, d)
    np.testing.assert_array_equal(H2.to_dense(), H.to_dense())
    assert d["bl_rank"].sum() == sum(H.ranks().values())
