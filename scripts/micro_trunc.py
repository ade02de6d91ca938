"""Latency of the batched TRUNC for a batch of identical random low-rank-ish stacks."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_1703_09085_b200 as hm
ctx = hm.Context(0)
rng = np.random.default_rng(0)
for (m, n, l, r) in [(32, 32, 16, 8), (64, 64, 24, 10), (64, 64, 64, 20), (128, 128, 40, 15), (128, 128, 128, 40),
                     (256, 256, 60, 20), (64, 512, 40, 15), (500, 500, 100, 30)]:
    A = rng.standard_normal((m, r)) @ rng.standard_normal((r, l))
    B = rng.standard_normal((n, l))
    for nb in (1, 148):
        stacks = [(A, B)] * nb
        hm.test_trunc_batched(ctx, stacks, 1e-6)
        t = time.time()
        for _ in range(5):
            hm.test_trunc_batched(ctx, stacks, 1e-6)
        dt = (time.time() - t) / 5
        print(f"m={m} n={n} l={l} r={r} batch={nb}: {dt*1e3:.2f} ms per call (incl. upload/sync)")
ctx.profile(True)
for (m, n, l, r) in [(64, 64, 24, 10), (128, 128, 40, 15)]:
    A = rng.standard_normal((m, r)) @ rng.standard_normal((r, l)); B = rng.standard_normal((n, l))
    ctx.profile_reset()
    for _ in range(10): hm.test_trunc_batched(ctx, [(A, B)], 1e-6)
    p = ctx.profile_get()
    print(m, n, l, {k: round(v['ms'] / max(v['launches'], 1), 4) for k, v in p.items() if v['launches']})
