#!/bin/bash
T=${TAG:-r1l}
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/${T}_pytest.log 2>&1; echo "pytest $?"; tail -2 $O/${T}_pytest.log
for v in "HM_X=0" "HM_QR_LAT512=0" "HM_TSQR_ROWS_LAT=768 HM_TSQR_H_LAT=384" "HM_QR_RB=8"; do
  env $v timeout 600 python scripts/prof_factor.py lr 6 64 1e-6 > "$O/${T}_prof_lr_${v// /_}.log" 2>&1; echo "prof $v $?"
done
timeout 300 python bench.py --no-factor --no-cpu-baseline --steps 2 --warmup 2 > "$O/${T}_bench.json" 2>&1; echo "bench $?"
