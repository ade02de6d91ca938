"""Latency / throughput of the staged TRUNC (QR classes) on batches of identical stacks; per-class ms."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_1703_09085_b200 as hm
ctx = hm.Context(0)
rng = np.random.default_rng(0)
ctx.profile(True)
for (m, n, l, r) in [(272, 69, 69, 30), (248, 120, 77, 30), (500, 480, 96, 35), (760, 700, 128, 40), (1400, 1300, 140, 40)]:
    A = rng.standard_normal((m, r)) @ rng.standard_normal((r, l)) * (10.0 ** (-0.3 * np.arange(l)))
    B = rng.standard_normal((n, l))
    for nb in (4, 592):
        stacks = [(A, B)] * nb
        hm.test_trunc_batched(ctx, stacks, 1e-6)
        ctx.profile_reset()
        for _ in range(3): hm.test_trunc_batched(ctx, stacks, 1e-6)
        p = ctx.profile_get()
        print(f"m={m} n={n} l={l} batch={nb}:", {k: round(v['ms'] / 3, 3) for k, v in p.items() if v['launches'] and v['ms'] > 0.001}, flush=True)
