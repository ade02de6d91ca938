#!/bin/bash
# One GPU session: parity tests, bench line, ncu launch list of one bench step
# and one full capture of the top kernel.  Usage (from the repo root, on a
# gpurun box):  bash scripts/gpu_round.sh TAG [KERNEL_REGEX] [LAUNCH_SKIP]
TAG=${1:-r1}
KREGEX=${2:-k_eval2}
KSKIP=${3:-3}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/${TAG}_smi.txt 2>&1
if [ -z "$SKIP_TESTS" ]; then
  timeout 1800 python -m pytest tests -m gpu -q > $OUT/${TAG}_pytest_gpu.log 2>&1
  echo "pytest exit $?" >> $OUT/${TAG}_pytest_gpu.log
  tail -3 $OUT/${TAG}_pytest_gpu.log
fi
if [ -z "$SKIP_BENCH" ]; then
  timeout 1500 python bench.py > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err
  echo "bench exit $?"
  tail -c 600 $OUT/${TAG}_bench.json
  timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > $OUT/${TAG}_bench_ref.json 2> $OUT/${TAG}_bench_ref.err
  echo "bench ref exit $?"
fi
if [ -z "$SKIP_NCU" ]; then
  timeout 600 python scripts/ncu_step.py save /tmp/cfg4.npz > $OUT/${TAG}_ncu_save.log 2>&1
  timeout 1200 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $OUT/${TAG}_launches.csv python scripts/ncu_step.py load /tmp/cfg4.npz > $OUT/${TAG}_ncu_list.log 2>&1
  echo "ncu list exit $?"
  python scripts/ncu_summary.py $OUT/${TAG}_launches.csv > $OUT/${TAG}_launches_summary.md 2>&1
  head -20 $OUT/${TAG}_launches_summary.md
  timeout 1200 ncu --profile-from-start off --set full --clock-control none --import-source on \
      -k regex:"$KREGEX" --launch-skip $KSKIP -c 1 -o $OUT/${TAG}_${KREGEX//[^a-zA-Z0-9_]/}_full \
      python scripts/ncu_step.py load /tmp/cfg4.npz > $OUT/${TAG}_ncu_full.log 2>&1
  echo "ncu full exit $?"
fi
