#!/bin/bash
# A/B timings of the scheduler knobs (one gpurun call): merged vs serial
# factorization recursion, auxiliary streams on / off.  Usage: bash scripts/gpu_ab.sh TAG
TAG=${1:-ab}
OUT=gpurun_out; mkdir -p $OUT
{
timeout 900 python -m pytest tests/test_gpu_factor.py tests/test_gpu_golden.py -m gpu -q -x 2>&1 | tail -15
echo "== H-LR n=81920 merged"
HM_DEBUG_TIMING=1 timeout 600 python scripts/time_factor.py lr 6 64 1e-6 2 2>&1 | tail -4
echo "== H-LR n=81920 serial"
HM_FACTOR_SERIAL=1 HM_DEBUG_TIMING=1 timeout 600 python scripts/time_factor.py lr 6 64 1e-6 1 2>&1 | tail -3
echo "== H-Chol n=20480 merged"
HM_DEBUG_TIMING=1 timeout 600 python scripts/time_factor.py chol 5 32 1e-5 2 2>&1 | tail -4
echo "== product cfg4 streams on"
timeout 600 python scripts/time_addmul.py 6 64 1e-6 4 2>&1 | tail -4
echo "== product cfg4 streams off"
HM_STREAMS=0 timeout 600 python scripts/time_addmul.py 6 64 1e-6 4 2>&1 | tail -4
} > $OUT/${TAG}_ab.log 2>&1
cat $OUT/${TAG}_ab.log
