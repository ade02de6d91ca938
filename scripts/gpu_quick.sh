#!/bin/bash
# Quick effect check: trunc-kernel parity, micro QR, H-LR n=20480 / n=81920, config-4 product.
TAG=${1:-q}
OUT=gpurun_out; mkdir -p $OUT
{
python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "trunc_kernel" 2>&1 | tail -2
python scripts/micro_qr.py 2>&1
HM_DEBUG_TIMING=1 timeout 300 python scripts/time_factor.py lr 5 64 1e-6 2 2>&1 | grep "^lr\|hm_factor" | tail -2
HM_DEBUG_TIMING=1 timeout 600 python scripts/time_factor.py lr 6 64 1e-6 2 2>&1 | grep "^lr\|hm_factor" | tail -2
timeout 600 python scripts/time_addmul.py 6 64 1e-6 4 2>&1 | tail -3
} > $OUT/${TAG}_quick.log 2>&1
cat $OUT/${TAG}_quick.log
