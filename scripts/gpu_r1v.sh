#!/bin/bash
O=gpurun_out
mkdir -p $O
timeout 1200 python scripts/time_factor.py lr 7 64 1e-4 1 > $O/r1v_hlr_cfg5.log 2>&1; echo "cfg5 $?"; tail -3 $O/r1v_hlr_cfg5.log
