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
python /tmp/tiny.py 5 64 > $OUT/np3_plain5.log 2>&1; echo "plain5 $?"; cat $OUT/np3_plain5.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 5 --csv --log-file $OUT/np3_l5.csv python /tmp/tiny.py 5 64 > $OUT/np3_l5.log 2>&1
echo "L5 exit $?"; tail -3 $OUT/np3_l5.log
HM_NO_PRESUM=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 5 --csv --log-file $OUT/np3_l5np.csv python /tmp/tiny.py 5 64 > $OUT/np3_l5np.log 2>&1
echo "L5 nopresum exit $?"; tail -3 $OUT/np3_l5np.log
