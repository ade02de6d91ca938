#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT
cat > /tmp/tiny.py <<'PY'
import sys, time
sys.path.insert(0, '.')
import torch
import paper_1703_09085_b200 as hm
from hm_inputs import sphere_points
t0 = time.time()
ctx = hm.Context(0)
x, w = sphere_points(int(sys.argv[1]))
G = ctx.build(x, w, int(sys.argv[2]), 2.0, 1e-4)
print(f"built {time.time()-t0:.1f}", flush=True)
X, Y, Z = G.clone(), G.clone(), G.clone()
hm.addmul(1.0, X, Y, Z, 1e-4)
torch.cuda.synchronize()
print(f"addmul done {time.time()-t0:.1f} launches {ctx.last_stats()['kernel_launches']}", flush=True)
PY
python /tmp/tiny.py 2 8 > $OUT/np2_plain.log 2>&1 && echo plain ok
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/np2_tiny.csv python /tmp/tiny.py 2 8 > $OUT/np2_tiny.log 2>&1
echo "tiny exit $? $(wc -l < $OUT/np2_tiny.csv)"
HM_NO_PRESUM=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/np2_nopresum.csv python /tmp/tiny.py 2 8 > $OUT/np2_nopresum.log 2>&1
echo "tiny nopresum exit $? $(wc -l < $OUT/np2_nopresum.csv)"
