"""Reproduce a failing TRUNC stack alone / replicated (diagnostics)."""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_1703_09085_b200 as hm
ctx = hm.Context(0)
rng = np.random.default_rng(5)
m, n, l, r = 50, 700, 40, 20
# regenerate the generator stream of dbg_trunc3 up to this shape
for (mm, nn, ll, rr) in [(64, 64, 40, 20), (32, 32, 30, 10), (100, 90, 70, 30), (128, 128, 100, 60), (300, 280, 120, 80),
                         (600, 500, 300, 280), (400, 400, 350, 300)]:
    for nb in (1, 300):
        for _ in range(min(nb, 300 if mm * nn < 2e5 else 4)):
            rng.standard_normal((mm, rr)); rng.standard_normal((rr, ll)); rng.standard_normal((nn, ll))
stacks = []
for nb in (1, 300):
    for _ in range(nb):
        A = rng.standard_normal((m, r)) @ np.diag(10.0 ** (-0.1 * np.arange(r))) @ rng.standard_normal((r, l))
        B = rng.standard_normal((n, l))
        stacks.append((A, B))
bad = stacks[1 + 14]
def err(st, eps=1e-4):
    out, ranks, sig = hm.test_trunc_batched(ctx, st, eps)
    res = []
    for (A, B), (U, V), k, sg in zip(st, out, ranks, sig):
        M = A @ B.T
        res.append((int(k), float(np.linalg.norm(M - U @ V.T) / np.linalg.norm(M)), sg[:3], sg[19:23]))
    return res
print("alone", err([bad]))
print("x300", err([bad] * 300)[:2])
print("x300 other", err([stacks[1]] * 300)[:1])
np.savez("gpurun_out/bad_stack.npz", A=bad[0], B=bad[1])
s = np.linalg.svd(bad[0] @ bad[1].T, compute_uv=False)
print("numpy sigma", s[:3], s[19:23])
