import numpy as np, sys
sys.path.insert(0, '.')
import paper_1703_09085_b200 as hm
from oracle.lowrank import TruncCtx, trunc
from tests.hm_compare import lowrank_diff, lowrank_norm
ctx = hm.Context(0)
rng = np.random.default_rng(5)
stacks = []
for it in range(400):
    m, n = rng.integers(1, 60, size=2)
    l = int(rng.integers(0, 80))
    r = int(rng.integers(0, l + 1))
    A = rng.standard_normal((m, r)) @ rng.standard_normal((r, l)) if r else np.zeros((m, l))
    B = rng.standard_normal((n, l))
    if it % 3 == 0 and l >= 2:
        B[:, 1] = B[:, 0]; A[:, 1] = -A[:, 0]
    stacks.append((A, B))
for eps in [0.0, 1e-3]:
    out, ranks, sig = hm.test_trunc_batched(ctx, stacks, eps)
    nbad = 0
    for i, ((A, B), (U, V), k) in enumerate(zip(stacks, out, ranks)):
        Uo, Vo = trunc(A, B, TruncCtx(eps))
        d = lowrank_diff(U, V, Uo, Vo) / max(lowrank_norm(Uo, Vo), 1e-300)
        sv = np.linalg.svd(A @ B.T, compute_uv=False) if min(A.shape[0], B.shape[0]) else np.zeros(0)
        if (k != Uo.shape[1] and eps > 0) or (d > 1e-9 and np.linalg.norm(A@B.T) > 1e-12):
            nbad += 1
            if nbad < 15:
                print("BAD", i, A.shape, B.shape, "k", k, Uo.shape[1], "d", d, "sigmax err", np.abs(sig[i][:len(sv)] - sv[:len(sig[i])]).max() if len(sv) else 0)
    print("eps", eps, "bad", nbad)
