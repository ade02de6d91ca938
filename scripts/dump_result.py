"""Diagnostics: run one device operation and save the exported result
(hm_export host description) to gpurun_out/<name>.npz for an exact host-side
comparison with the oracle's raw result (.golden_raw/)."""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_1703_09085_b200 as hm
from hm_inputs import sphere_points
what, L, leaf, eps, out = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), float(sys.argv[4]), sys.argv[5]
ctx = hm.Context(0)
x, w = sphere_points(L)
G = ctx.build(x, w, leaf, 2.0, eps, kernel=1 if what == "chol" else 0)
if what == "product":
    X, Y, Z = G.clone(), G.clone(), G.clone()
    hm.addmul(1.0, X, Y, Z, eps)
    R = Z
elif what == "lr":
    hm.lr(G, eps); R = G
else:
    hm.chol(G, eps); R = G
d = R.export()
np.savez_compressed(out, **{k: v for k, v in d.items() if v is not None})
print("saved", out, ctx.last_stats()["truncations"])
