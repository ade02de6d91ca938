#!/bin/bash
T=${TAG:-r1q}
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/${T}_pytest.log 2>&1; echo "pytest $?"; tail -2 $O/${T}_pytest.log
for v in "HM_X=0" "HM_QR_DMMA=0"; do
  env $v timeout 300 python bench.py --no-factor --no-cpu-baseline --steps 2 --warmup 2 > "$O/${T}_bench_${v// /_}.json" 2>&1; echo "$v $?"
  env $v timeout 600 python scripts/prof_factor.py lr 6 64 1e-6 > "$O/${T}_prof_lr_${v// /_}.log" 2>&1; echo "prof $v $?"
done
