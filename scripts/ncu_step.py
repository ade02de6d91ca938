"""One hm_addmul step (config 4) bracketed by cudaProfilerStart/Stop, for
`ncu --profile-from-start off` launch lists / full captures of the bench step."""
import sys
sys.path.insert(0, '.')
import torch
import paper_1703_09085_b200 as hm
from hm_inputs import sphere_points
L, leaf, eps = (int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3])) if len(sys.argv) > 3 else (6, 64, 1e-6)
ctx = hm.Context(0)
x, w = sphere_points(L)
G = ctx.build(x, w, leaf, 2.0, eps)
X, Y = G.clone(), G.clone()
Z = G.clone()
hm.addmul(1.0, X, Y, Z, eps)          # warm-up (pools, caches)
Z.free()
Z = G.clone()
torch.cuda.synchronize()
print("launches before step:", ctx.last_stats()["kernel_launches"], flush=True)
torch.cuda.profiler.start()
hm.addmul(1.0, X, Y, Z, eps)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("launches in step:", ctx.last_stats()["kernel_launches"])
