"""S0 (standard, hm_addmul_std) vs S2 (accumulated, hm_addmul) on one config:
device time (CUDA events), truncation counts, rounds, peak memory; the
paper's central comparison (Fig. 9).
    python scripts/time_std.py L leaf eps"""
import sys, time
sys.path.insert(0, '.')
import torch
import paper_1703_09085_b200 as hm
from hm_inputs import sphere_points
L, leaf, eps = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3])
ctx = hm.Context(0)
x, w = sphere_points(L)
G = ctx.build(x, w, leaf, 2.0, eps)
X, Y = G.clone(), G.clone()
st = torch.cuda.current_stream()
for name, fn in (("S2", hm.addmul), ("S0", hm.addmul_std), ("S2", hm.addmul), ("S0", hm.addmul_std)):
    Z = G.clone()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    fn(1.0, X, Y, Z, eps)
    e1.record(st)
    torch.cuda.synchronize()
    s = ctx.last_stats()
    print(f"{name} n={len(w)} {e0.elapsed_time(e1) / 1e3:.3f}s truncations {s['truncations']} trunc_cols {s['trunc_cols']} "
          f"rounds/levels {s['levels']} gflop {(s['flops_trunc'] + s['flops_eval'] + s['flops_dense']) / 1e9:.1f}", flush=True)
    Z.free()
