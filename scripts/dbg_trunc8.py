"""SVD of the dumped M through the fused kernel and through k_svd (diagnostics)."""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_1703_09085_b200 as hm
ctx = hm.Context(0)
M = np.load("dbg/M.npy")
A = np.hstack([M, np.zeros((50, 10))])
B = np.zeros((40, 50)); B[:, :40] = np.eye(40)
for st in [(A, B), (M.T.copy(), np.eye(50))]:
    out, ranks, sig = hm.test_trunc_batched(ctx, [st], 1e-4)
    U, V = out[0]
    MM = st[0] @ st[1].T
    print(st[0].shape, st[1].shape, int(ranks[0]), np.linalg.norm(MM - U @ V.T) / np.linalg.norm(MM), sig[0][:3])
