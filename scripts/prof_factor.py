"""Diagnostics: device H-LR / H-Cholesky time at a config (+ probe residual)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_1703_09085_b200 as hm
from hm_inputs import sphere_points, probe_vectors
kind, L, leaf, eps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), float(sys.argv[4])
ctx = hm.Context(0)
x, w = sphere_points(L)
t = time.time(); G = ctx.build(x, w, leaf, 2.0, eps, kernel=0 if kind == "lr" else 1); tb = time.time() - t
G0 = G.clone()
ctx.profile(True); ctx.profile_reset()
torch.cuda.synchronize()
t = time.time()
(hm.lr if kind == "lr" else hm.chol)(G, eps)
torch.cuda.synchronize()
dt = time.time() - t
st = ctx.last_stats()
print(f"{kind} n={len(w)} build {tb:.2f}s factor {dt:.3f}s trunc {st['truncations']} flushes {st['levels']} launches? min_pivot {st['min_pivot']:.3e}")
for k, v in sorted(ctx.profile_get().items(), key=lambda kv: -kv[1]["ms"])[:8]:
    if v["launches"]: print(f"  {k:14s} {v['ms']:10.1f} ms {v['launches']:7d} launches")
