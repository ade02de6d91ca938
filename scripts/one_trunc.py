"""One single-stack TRUNC at shape (m, n, l) with a kernel-like spectrum (for ncu captures)."""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_1703_09085_b200 as hm
m, n, l = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
decay = float(sys.argv[4]) if len(sys.argv) > 4 else 0.15
ctx = hm.Context(0)
rng = np.random.default_rng(0)
q = min(m, n, l)
s = 10.0 ** (-decay * np.arange(q))
U, _ = np.linalg.qr(rng.standard_normal((m, q)))
V, _ = np.linalg.qr(rng.standard_normal((n, q)))
A = np.hstack([U * s, (U * s) @ rng.standard_normal((q, l - q))]) if l > q else U * s
B = np.hstack([V, np.zeros((n, l - q))]) if l > q else V
for _ in range(2):
    out, ranks, _ = hm.test_trunc_batched(ctx, [(A, B)], 1e-6)
print("rank", ranks[0])
