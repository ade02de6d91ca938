#!/bin/bash
# parity subset + bench variants (QR occupancy, TSQR threshold)
T=${TAG:-r1h}
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/${T}_pytest.log 2>&1; echo "pytest $?"; tail -2 $O/${T}_pytest.log
for v in "HM_X=0" "HM_QR_OCC3=0" "HM_TSQR_ROWS=768 HM_TSQR_H=384" "HM_TSQR_ROWS=1024 HM_TSQR_H=512"; do
  env $v timeout 300 python bench.py --no-factor --no-cpu-baseline --steps 2 --warmup 2 > "$O/${T}_bench_${v// /_}.json" 2>&1; echo "$v $?"
done
