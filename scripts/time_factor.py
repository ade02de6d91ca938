"""Wall-clock of device H-LR / H-Cholesky (no profiling)."""
import sys, time
sys.path.insert(0, '.')
import torch
import paper_1703_09085_b200 as hm
from hm_inputs import sphere_points
kind, L, leaf, eps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), float(sys.argv[4])
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 2
ctx = hm.Context(0)
x, w = sphere_points(L)
G0 = ctx.build(x, w, leaf, 2.0, eps, kernel=0 if kind == "lr" else 1)
for r in range(reps):
    G = G0.clone()
    torch.cuda.synchronize(); t = time.time()
    (hm.lr if kind == "lr" else hm.chol)(G, eps)
    torch.cuda.synchronize(); dt = time.time() - t
    st = ctx.last_stats()
    print(f"{kind} n={len(w)} factor {dt:.3f}s trunc {st['truncations']} flushes {st['levels']} min_pivot {st['min_pivot']:.3e}", flush=True)
    G.free()
