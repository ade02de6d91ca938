"""Dump the SVD input M of the failing stack, then TRUNC(M, I) (diagnostics)."""
import os, sys
sys.path.insert(0, '.')
import numpy as np
import paper_1703_09085_b200 as hm
ctx = hm.Context(0)
d = np.load("gpurun_out/bad_stack.npz")
A, B = d["A"], d["B"]
os.environ["HM_DUMP_M"] = "gpurun_out/M.bin"
hm.test_trunc_batched(ctx, [(A, B)], 1e-4)
M = np.fromfile("gpurun_out/M.bin").reshape((40, 50)).T   # tall orientation 50 x 40, column-major
np.save("gpurun_out/M.npy", M)
out, ranks, sig = hm.test_trunc_batched(ctx, [(M, np.eye(40))], 1e-4)
U, V = out[0]
print("TRUNC(M, I):", int(ranks[0]), np.linalg.norm(M - U @ V.T) / np.linalg.norm(M), sig[0][:3], np.linalg.svd(M, compute_uv=False)[:3])
