"""Batched TRUNC check at many shapes and batch sizes (256- and 512-thread paths)."""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_1703_09085_b200 as hm
ctx = hm.Context(0)
rng = np.random.default_rng(5)
def check(stacks, eps):
    out, ranks, sig = hm.test_trunc_batched(ctx, stacks, eps)
    bad = []
    for idx, ((A, B), (U, V), k) in enumerate(zip(stacks, out, ranks)):
        M = A @ B.T
        s = np.linalg.svd(M, compute_uv=False)
        tot = np.sum(s ** 2)
        kk = next(j for j in range(len(s) + 1) if np.sum(s[j:] ** 2) <= eps ** 2 * tot)
        err = np.linalg.norm(M - U @ V.T) / max(np.linalg.norm(M), 1e-300)
        ref = np.sqrt(np.sum(s[kk:] ** 2)) / max(np.sqrt(tot), 1e-300)
        if eps == 0.0:
            ok = err <= 1e-12 * np.sqrt(len(s))
        else:
            ok = k == kk and abs(err - ref) <= 1e-8 + 1e-6 * ref
        if not ok:
            bad.append((idx, A.shape[0], B.shape[0], A.shape[1], k, kk, err, ref))
    return bad
for (m, n, l, r) in [(64, 64, 40, 20), (32, 32, 30, 10), (100, 90, 70, 30), (128, 128, 100, 60), (300, 280, 120, 80),
                     (600, 500, 300, 280), (400, 400, 350, 300), (50, 700, 40, 20), (1000, 900, 300, 150)]:
    for nb in (1, 300):
        stacks = []
        for _ in range(min(nb, 300 if m * n < 2e5 else 4)):
            A = rng.standard_normal((m, r)) @ np.diag(10.0 ** (-0.1 * np.arange(r))) @ rng.standard_normal((r, l))
            B = rng.standard_normal((n, l))
            stacks.append((A, B))
        for eps in (1e-4, 0.0):
            bad = check(stacks, eps)
            print(m, n, l, r, "batch", len(stacks), "eps", eps, "bad", len(bad), bad[:2], flush=True)
