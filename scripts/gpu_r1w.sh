#!/bin/bash
T=r1w
O=gpurun_out
mkdir -p $O
for v in "HM_X=0" "HM_EVAL_SPLIT=4736" "HM_EVAL_SPLIT=18944"; do
  env $v timeout 300 python bench.py --no-factor --no-cpu-baseline --steps 2 --warmup 2 > "$O/${T}_bench_${v// /_}.json" 2>&1; echo "$v $?"
done
