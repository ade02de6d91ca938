#!/bin/bash
# A/B of the TSQR chunking (even chunks, row threshold) on the config-4 product and the H-LR.
TAG=${1:-tsqr}
OUT=gpurun_out; mkdir -p $OUT
{
python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "trunc_kernel" 2>&1 | tail -2
run() { echo "== $*"; env "$@" timeout 600 python scripts/time_addmul.py 6 64 1e-6 3 2>&1 | tail -1; env "$@" timeout 300 python scripts/time_factor.py lr 5 64 1e-6 2 2>&1 | grep "^lr" | tail -1; }
run X=1
run HM_TSQR_EVEN=0
run HM_TSQR_ROWS=768 HM_TSQR_ROWS_LAT=768
run HM_TSQR_ROWS=768 HM_TSQR_ROWS_LAT=768 HM_TSQR_H=384 HM_TSQR_H_LAT=384
run HM_TSQR_ROWS=1024 HM_TSQR_ROWS_LAT=1024
HM_TSQR_ROWS=768 HM_TSQR_ROWS_LAT=768 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "trunc_kernel" 2>&1 | tail -2
} > $OUT/${TAG}_tsqr.log 2>&1
cat $OUT/${TAG}_tsqr.log
