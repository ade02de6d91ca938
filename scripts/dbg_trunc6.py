"""Failing-stack check under the current env (diagnostics)."""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_1703_09085_b200 as hm
ctx = hm.Context(0)
d = np.load("gpurun_out/bad_stack.npz")
A, B = d["A"], d["B"]
for name, st in [("A,B", (A, B)), ("A,-B", (A, -B)), ("2A,B", (2 * A, B)), ("A,B[:,perm]", (A[:, ::-1], B[:, ::-1]))]:
    out, ranks, sig = hm.test_trunc_batched(ctx, [st], 1e-4)
    U, V = out[0]
    M = st[0] @ st[1].T
    print(name, int(ranks[0]), np.linalg.norm(M - U @ V.T) / np.linalg.norm(M), sig[0][:2])
