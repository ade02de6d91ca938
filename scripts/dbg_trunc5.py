"""Bisect a failing TRUNC stack: QR of B vs SVD (diagnostics)."""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_1703_09085_b200 as hm
ctx = hm.Context(0)
d = np.load("gpurun_out/bad_stack.npz")
A, B = d["A"], d["B"]
R = np.linalg.qr(B, mode="r")
for name, st in [("A,B", (A, B)), ("A,R_B", (A, R)), ("A,B[:600]", (A[:, :], B[:600])), ("A,B[:500]", (A, B[:500]))]:
    out, ranks, sig = hm.test_trunc_batched(ctx, [st], 1e-4)
    U, V = out[0]
    M = st[0] @ st[1].T
    print(name, int(ranks[0]), np.linalg.norm(M - U @ V.T) / np.linalg.norm(M), sig[0][:2], np.linalg.svd(M, compute_uv=False)[:2])
