#!/bin/bash
# bench variants: fused-TRUNC 26K bucket threads, global SVD threads
T=${TAG:-r1i}
O=gpurun_out
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py -k "addmul or product or trunc" -x -q > $O/${T}_pytest.log 2>&1; echo "pytest $?"; tail -2 $O/${T}_pytest.log
for v in "HM_X=0" "HM_TS26_THREADS=256" "HM_SVDG_THREADS=256" "HM_SVDG_THREADS=256 HM_QR_OCC3=0"; do
  env $v timeout 300 python bench.py --no-factor --no-cpu-baseline --steps 2 --warmup 2 > "$O/${T}_bench_${v// /_}.json" 2>&1; echo "$v $?"
done
timeout 600 python scripts/prof_factor.py lr 6 64 1e-6 > $O/${T}_prof_lr.log 2>&1; echo "prof lr $?"
