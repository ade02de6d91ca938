"""Small device runs for compute-sanitizer (memcheck / racecheck / synccheck):
the product (S2 and S0), H-LR, H-Cholesky, inversion and solves at n = 320
(leaf 8) and the product + H-LR at n = 1280 (config 1), all through the C-ABI."""
import sys
sys.path.insert(0, '.')
import torch
import paper_1703_09085_b200 as hm
from hm_inputs import sphere_points
ctx = hm.Context(0)
for L, leaf, eps in [(2, 8, 1e-4), (3, 32, 1e-4)]:
    x, w = sphere_points(L)
    G = ctx.build(x, w, leaf, 2.0, eps)
    X, Y, Z = G.clone(), G.clone(), G.clone()
    hm.addmul(1.0, X, Y, Z, eps)
    Z2 = G.clone()
    hm.addmul_std(1.0, X, Y, Z2, eps)
    F = G.clone()
    hm.lr(F, eps)
    v = torch.randn(len(w), 2, dtype=torch.float64, device="cuda").T.contiguous().T
    hm.solve(F, v, "L")
    hm.solve(F, v, "R")
    if L == 2:
        Gs = ctx.build(x, w, leaf, 2.0, eps, kernel=1)
        hm.chol(Gs, eps)
        Gi = G.clone()
        hm.inv(Gi, eps)
    torch.cuda.synchronize()
    print(f"n={len(w)} ok: truncations {ctx.last_stats()['truncations']}", flush=True)
print("sanitize case done")
