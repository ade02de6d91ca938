"""Diagnostics: hm_addmul at a config with per-class timing (+ optional job dump)."""
import json, os, sys, time
sys.path.insert(0, '.')
import torch
import paper_1703_09085_b200 as hm
from hm_inputs import sphere_points
L, leaf, eps = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 2
ctx = hm.Context(0)
x, w = sphere_points(L)
t = time.time(); G = ctx.build(x, w, leaf, 2.0, eps); print("build", time.time() - t, flush=True)
X, Y = G.clone(), G.clone()
for r in range(reps):
    Z = G.clone()
    ctx.profile(True); ctx.profile_reset()
    t = time.time(); hm.addmul(1.0, X, Y, Z, eps); dt = time.time() - t
    print("addmul s", dt, flush=True)
    Z.free()
print(ctx.last_stats())
for k, v in sorted(ctx.profile_get().items(), key=lambda kv: -kv[1]["ms"]):
    if v["launches"]: print(f"{k:14s} {v['ms']:10.1f} ms  {v['launches']:5d} launches  {v['flops']/1e9:10.1f} GF  {v['bytes']/1e9:8.2f} GB(or jobs)")
