#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck; one tool per run) on the
# small C-ABI cases of scripts/sanitize_case.py.  Usage: bash scripts/gpu_sanitize.sh TAG
TAG=${1:-san}
OUT=gpurun_out; mkdir -p $OUT
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 1500 $CS --tool $tool --print-limit 20 python scripts/sanitize_case.py > $OUT/${TAG}_sanitize_${tool}.log 2>&1
  echo "$tool exit $?" >> $OUT/${TAG}_sanitize_${tool}.log
  tail -4 $OUT/${TAG}_sanitize_${tool}.log
done
