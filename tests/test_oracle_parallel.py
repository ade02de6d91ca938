"""Pin of oracle/parallel.py (the drivers that wrote the full-size goldens):
build_parallel and addmul_s2_parallel must be BIT-IDENTICAL to the serial
oracle (oracle.hmatrix.build, oracle.product.addmul_s2) -- same truncation
inputs in the same order inside every independent subtree (Parallelization
remark P:L1330-1336), hence the same floating-point results -- with the same
truncation / addproduct counts."""
import os

import numpy as np
import pytest

from hm_inputs import sphere_points
from oracle.hmatrix import Problem, build
from oracle.lowrank import TruncCtx
from oracle.parallel import addmul_s2_parallel, build_parallel
from oracle.product import addmul_s2

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")


def _identical(h1, h2):
    assert h1.A.keys() == h2.A.keys() and h1.N.keys() == h2.N.keys()
    for k in h1.A:
        assert np.array_equal(h1.A[k], h2.A[k]) and np.array_equal(h1.B[k], h2.B[k]), k
    for k in h1.N:
        assert np.array_equal(h1.N[k], h2.N[k]), k


@pytest.mark.parametrize("L,leaf,eps,depth", [(3, 32, 1e-4, 3), (3, 16, 1e-6, 4)])
def test_parallel_oracle_bit_identical(L, leaf, eps, depth):
    x, w = sphere_points(L)
    P = Problem(x, w, leaf, 2.0)
    G = build(P, eps)
    Gp = build_parallel(P, eps, workers=4)
    _identical(G, Gp)
    ctx = TruncCtx(eps)
    Zs, ctx, st = addmul_s2(1.0, G.clone(), G.clone(), G.clone(), eps, ctx=ctx)
    Zp, info = addmul_s2_parallel(1.0, G.clone(), G.clone(), G.clone(), eps, workers=4, frontier_depth=depth)
    _identical(Zs, Zp)
    assert info["truncations"] == ctx.count
    assert info["trunc_cols"] == ctx.cols
    assert info["addproduct"] == st.addproduct
    assert sorted(map(str, (t for t, _ in info["near"]))) == sorted(map(str, (e[1] for e in ctx.near)))
