#!/bin/bash
# Per-launch-group timelines (HM_PROF_LOG) of the H-LR at n=20480 / n=81920 and
# of the config-4 product.  Usage: bash scripts/gpu_plog.sh TAG
TAG=${1:-plog}
OUT=gpurun_out; mkdir -p $OUT
HM_DEBUG_TIMING=1 HM_PROF_LOG=$OUT/${TAG}_hlr_L5.plog timeout 600 python scripts/prof_factor.py lr 5 64 1e-6 > $OUT/${TAG}_hlr_L5.log 2>&1
HM_DEBUG_TIMING=1 HM_PROF_LOG=$OUT/${TAG}_hlr_L6.plog timeout 900 python scripts/prof_factor.py lr 6 64 1e-6 > $OUT/${TAG}_hlr_L6.log 2>&1
HM_STREAMS=0 HM_PROF_LOG=$OUT/${TAG}_prod_L6.plog timeout 900 python scripts/prof_addmul.py 6 64 1e-6 2 > $OUT/${TAG}_prod_L6.log 2>&1
HM_STREAMS=0 HM_QR_STEPPED=0 timeout 900 python scripts/prof_addmul.py 6 64 1e-6 2 > $OUT/${TAG}_prod_L6_nostep.log 2>&1
gzip -f $OUT/${TAG}_*.plog
tail -12 $OUT/${TAG}_hlr_L6.log
tail -30 $OUT/${TAG}_prod_L6.log
tail -30 $OUT/${TAG}_prod_L6_nostep.log
