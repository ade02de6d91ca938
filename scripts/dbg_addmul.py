import numpy as np, sys, os
sys.path.insert(0, '.')
import paper_1703_09085_b200 as hm
from hm_inputs import sphere_points
from oracle.hmatrix import Problem, build, export
from oracle.lowrank import TruncCtx
from oracle.product import addmul_s2
from tests.hm_compare import leaf_payloads, lowrank_diff, lowrank_norm
L, leaf, eps = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3])
x, w = sphere_points(L)
P = Problem(x, w, leaf, 2.0)
G = build(P, eps)
Zo, octx, st = addmul_s2(1.0, G.clone(), G.clone(), G.clone(), eps, ctx=TruncCtx(eps))
ctx = hm.Context(0)
Gg = ctx.import_desc(export(G))
X, Y, Z = Gg.clone(), Gg.clone(), Gg.clone()
try:
    hm.addmul(1.0, X, Y, Z, eps)
except Exception as e:
    print("ERR", e); raise
dg = Z.export(); do = export(Zo)
pg, po = leaf_payloads(dg), leaf_payloads(do)
bad = []
for b, vo in po.items():
    vg = pg[b]
    if vo[0] == 'dense':
        rel = np.linalg.norm(vg[1]-vo[1])/max(np.linalg.norm(vo[1]),1e-300)
    else:
        rel = lowrank_diff(vg[1], vg[2], vo[1], vo[2])/max(lowrank_norm(vo[1],vo[2]),1e-300)
    if rel > 1e-9:
        blk = P.bt.blocks[b]
        bad.append((b, vo[0], blk.level, blk.t.size, blk.s.size, rel))
print("bad", len(bad), "of", len(po))
for r in bad[:30]: print(r)
# which oracle flush branch: look at tags
tags = {}
for tag, k in octx.ranks:
    tags.setdefault((tag[0],) if tag else None, 0)
print(ctx.last_stats())
for (b, kind, lev, m, n, rel) in bad:
    blk = P.bt.blocks[b]
    t, r = blk.t, blk.s
    print("block", b, "t", t.id, t.size, "leaf" if t.leaf else "", "r", r.id, r.size, "leaf" if r.leaf else "")
    for tag, k in octx.ranks:
        if tag and tag[1:] == (t.id, r.id): print("   ", tag, k)
    # sons tags
    for ts in t.sons:
        for rs in r.sons:
            for tag, k in octx.ranks:
                if tag and tag[1:] == (ts.id, rs.id): print("      son", tag, k)
