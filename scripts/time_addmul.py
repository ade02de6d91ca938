"""Wall-clock of device hm_addmul (no profiling): python scripts/time_addmul.py L leaf eps [reps]."""
import sys, time
sys.path.insert(0, '.')
import torch
import paper_1703_09085_b200 as hm
from hm_inputs import sphere_points
L, leaf, eps = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
ctx = hm.Context(0)
x, w = sphere_points(L)
G = ctx.build(x, w, leaf, 2.0, eps)
X, Y = G.clone(), G.clone()
for r in range(reps):
    Z = G.clone()
    torch.cuda.synchronize(); t = time.time()
    hm.addmul(1.0, X, Y, Z, eps)
    torch.cuda.synchronize(); dt = time.time() - t
    st = ctx.last_stats()
    print(f"addmul n={len(w)} {dt:.3f}s trunc {st['truncations']} launches {st['kernel_launches']}", flush=True)
    Z.free()
