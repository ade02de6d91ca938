"""One hm_addmul step (config 4) bracketed by cudaProfilerStart/Stop, for
`ncu --profile-from-start off` launch lists / full captures of the bench step.

    python scripts/ncu_step.py save PATH     build config 4 and save its host description
    python scripts/ncu_step.py load PATH     import it (no build kernels: ncu's per-launch
                                             overhead would otherwise dominate), warm-up step,
                                             then ONE profiled step
"""
import sys
import time
T0 = time.time()
sys.path.insert(0, '.')
import numpy as np
import torch
import paper_1703_09085_b200 as hm
from hm_inputs import sphere_points
mode, path = sys.argv[1], sys.argv[2]
import os
# NCU_L: icosphere level (6 = config 4; ncu's per-launch overhead grows with the
# allocated device memory: the committed captures use L = 5, n = 20480, the
# same leaf / eta / eps and the same kernels at the deep levels)
L, leaf, eps = int(os.environ.get("NCU_L", "6")), 64, 1e-6
ctx = hm.Context(0)
if mode == "save":
    x, w = sphere_points(L)
    G = ctx.build(x, w, leaf, 2.0, eps)
    d = G.export()
    np.savez(path, **{k: v for k, v in d.items() if v is not None})
    print("saved", path)
    sys.exit(0)
z = np.load(path)
d = {k: z[k] for k in z.files}
d["perm"] = d.get("perm")
print(f"[{time.time()-T0:.1f}s] loaded npz", flush=True)
G = ctx.import_desc(d)
torch.cuda.synchronize()
print(f"[{time.time()-T0:.1f}s] imported", flush=True)
X, Y = G.clone(), G.clone()
Z = G.clone()
import os
if not os.environ.get("HM_NCU_NOWARM"):
    hm.addmul(1.0, X, Y, Z, eps)          # warm-up (pools, caches)
    torch.cuda.synchronize()
    print(f"[{time.time()-T0:.1f}s] warm-up step done", flush=True)
    Z.free()
    Z = G.clone()
torch.cuda.synchronize()
print("launches before step:", ctx.last_stats()["kernel_launches"], flush=True)
torch.cuda.profiler.start()
hm.addmul(1.0, X, Y, Z, eps)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print(f"[{time.time()-T0:.1f}s] launches after step:", ctx.last_stats()["kernel_launches"], flush=True)
