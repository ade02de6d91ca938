"""Timing of the end-to-end path: hm_import x3, hm_addmul, hm_export (config 4)."""
import sys, time
sys.path.insert(0, '.')
import torch
import paper_1703_09085_b200 as hm
from hm_inputs import sphere_points
ctx = hm.Context(0)
x, w = sphere_points(6)
G = ctx.build(x, w, 64, 2.0, 1e-6)
d = G.export()
if len(sys.argv) > 1 and sys.argv[1] == "pinned":
    for k in ("factors", "dense"):
        t = torch.empty(d[k].shape, dtype=torch.float64, pin_memory=True)
        t.numpy()[...] = d[k]
        d[k] = t.numpy()
for rep in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    Xh, Yh, Zh = ctx.import_desc(d), ctx.import_desc(d), ctx.import_desc(d)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    hm.addmul(1.0, Xh, Yh, Zh, 1e-6)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    out = Zh.export(pinned=len(sys.argv) > 1 and sys.argv[1] == "pinned")
    t3 = time.perf_counter()
    for m_ in (Xh, Yh, Zh):
        m_.free()
    print(f"import x3 {t1 - t0:.3f}s  addmul {t2 - t1:.3f}s  export {t3 - t2:.3f}s  total {t3 - t0:.3f}s", flush=True)
