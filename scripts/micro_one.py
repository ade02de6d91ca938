"""A few calls of the batched TRUNC on `batch` identical stacks (m, n, l, r) -- for ncu captures."""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_1703_09085_b200 as hm
m, n, l, r, batch = (int(a) for a in sys.argv[1:6])
ctx = hm.Context(0)
rng = np.random.default_rng(0)
A = rng.standard_normal((m, r)) @ rng.standard_normal((r, l)) * (10.0 ** (-0.3 * np.arange(l)))
B = rng.standard_normal((n, l))
for _ in range(3):
    out, ranks, _ = hm.test_trunc_batched(ctx, [(A, B)] * batch, 1e-6)
print("rank", ranks[0])
