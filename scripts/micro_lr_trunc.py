"""Latency of single-stack TRUNC at shapes typical of H-LR levels (kernel-like spectrum)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_1703_09085_b200 as hm
ctx = hm.Context(0)
rng = np.random.default_rng(0)
shapes = [(50, 53, 80), (120, 122, 16), (218, 218, 16), (64, 64, 64), (85, 400, 80), (100, 1000, 64), (205, 1500, 40)]
for (m, n, l) in shapes:
    q = min(m, n, l)
    s = 10.0 ** (-0.15 * np.arange(q))
    U, _ = np.linalg.qr(rng.standard_normal((m, q)))
    V, _ = np.linalg.qr(rng.standard_normal((n, q)))
    A = np.hstack([U * s, rng.standard_normal((m, l - q))]) if l > q else U * s
    B = np.hstack([V, np.zeros((n, l - q))]) if l > q else V
    hm.test_trunc_batched(ctx, [(A, B)], 1e-6)
    ctx.profile(True); ctx.profile_reset()
    for _ in range(5): hm.test_trunc_batched(ctx, [(A, B)], 1e-6)
    p = ctx.profile_get()
    ctx.profile(False)
    torch.cuda.synchronize(); t = time.time()
    for _ in range(5): hm.test_trunc_batched(ctx, [(A, B)], 1e-6)
    torch.cuda.synchronize(); dt = (time.time() - t) / 5
    print(f"m={m} n={n} l={l}: {dt*1e3:.3f} ms/call  " +
          " ".join(f"{k}={v['ms']/5:.3f}" for k, v in sorted(p.items(), key=lambda kv: -kv[1]['ms']) if v['launches']), flush=True)
