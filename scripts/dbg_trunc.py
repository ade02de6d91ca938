import numpy as np, sys
sys.path.insert(0, '.')
import paper_1703_09085_b200 as hm
from tests.test_gpu_parity import _prescribed
ctx = hm.Context(0)
rng = np.random.default_rng(12)
shapes = [(40, 30, 12, 0), (200, 150, 20, 2), (64, 64, 64, 1), (300, 40, 25, 3), (17, 500, 16, 2),
          (130, 170, 90, 4), (5, 3, 3, 0), (1, 1, 1, 0), (700, 650, 60, 3), (260, 240, 240, 2)]
stacks, svals = [], []
for m, n, q, junk in shapes:
    s = 10.0 ** (-np.arange(q) / 3.0)
    A, B = _prescribed(rng, m, n, s, junk)
    stacks.append((A, B)); svals.append(s)
for eps in [1e-4, 1e-6]:
    out, ranks, sig = hm.test_trunc_batched(ctx, stacks, eps)
    for (A,B),(U,V),k,s,sg,sh in zip(stacks,out,ranks,svals,sig,shapes):
        tot = np.sum(s**2)
        kk = next(j for j in range(len(s) + 1) if np.sum(s[j:] ** 2) <= eps ** 2 * tot)
        sv = np.linalg.svd(A@B.T, compute_uv=False)[:len(sg)]
        err = np.linalg.norm(A @ B.T - U @ V.T)
        print(sh, "k", k, "kk", kk, "sigerr", np.abs(sg[:len(s)]-s).max(), "vs np", np.abs(sg-sv).max(), "err", err, np.sqrt(np.sum(s[k:]**2)), "orth", np.abs(U.T@U-np.eye(k)).max() if k else 0)
