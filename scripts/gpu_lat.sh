#!/bin/bash
# A/B of the latency-mode thread counts on the H-LR (n = 20480, leaf 64, eps 1e-6).
TAG=${1:-lat}
OUT=gpurun_out; mkdir -p $OUT
{
run() { echo "== $*"; env "$@" HM_DEBUG_TIMING=1 timeout 300 python scripts/time_factor.py lr 5 64 1e-6 2 2>&1 | grep "^lr" | tail -1; }
run X=1
run HM_TS_LAT=256,256,256
run HM_TS_LAT=128,128,256
run HM_TS_LAT=128,128,128
run HM_TS_LAT=64,128,256
run HM_SVD_LAT=256
run HM_SVD_LAT=128
run HM_QR_LAT512=0
run HM_TS_LAT=128,128,256 HM_SVD_LAT=256 HM_QR_LAT512=0
} > $OUT/${TAG}_lat.log 2>&1
cat $OUT/${TAG}_lat.log
