import sys
sys.path.insert(0, '.')
import numpy as np
import paper_1703_09085_b200 as hm
from oracle.lowrank import TruncCtx, trunc
from tests.hm_compare import lowrank_diff, lowrank_norm
from tests.test_gpu_parity import _prescribed
ctx = hm.Context(0)
eps = 1e-6
rng = np.random.default_rng(2718)
shapes = []
for i in range(12):
    shapes.append((130 + 19 * i, 125 + 17 * i, 17 + 9 * i, i % 3))
    shapes.append((400 + 30 * i, 90 + 5 * i, 33 + 8 * i, i % 2))
    shapes.append((1600 + 400 * i, 300 + 20 * i, 20 + 6 * i, 1))
shapes += [(768, 767, 133, 0), (385, 384, 100, 1), (257, 256, 31, 2), (129, 128, 47, 0), (513, 512, 64, 1)]
stacks, svals = [], []
for m, n, q, junk in shapes:
    s = 10.0 ** (-0.21 * np.arange(q))
    A, B = _prescribed(rng, m, n, s, junk)
    stacks.append((A, B)); svals.append(s)
for mode in ("batch", "single"):
    if mode == "batch":
        out, ranks, _ = hm.test_trunc_batched(ctx, stacks, eps)
    else:
        out, ranks = [], []
        for st in stacks:
            o, r, _ = hm.test_trunc_batched(ctx, [st], eps)
            out.append(o[0]); ranks.append(r[0])
    for sh, (A, B), (U, V), k, s in zip(shapes, stacks, out, ranks, svals):
        kk = next(j for j in range(len(s) + 1) if np.sum(s[j:] ** 2) <= eps ** 2 * np.sum(s ** 2))
        Uo, Vo = trunc(A, B, TruncCtx(eps))
        d = lowrank_diff(U, V, Uo, Vo) / lowrank_norm(Uo, Vo) if k == Uo.shape[1] else -1
        flag = "" if (k == kk and 0 <= d <= 1e-9) else "  <<<<<<"
        print(mode, sh, "l", A.shape[1], "k", k, "kk", kk, "diff", f"{d:.2e}", flag)
