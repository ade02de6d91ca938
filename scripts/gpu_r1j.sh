#!/bin/bash
# parity tests + bench + variant benches + ncu launch list + one full capture
T=${TAG:-r1j}
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/${T}_pytest.log 2>&1; echo "pytest $?"; tail -2 $O/${T}_pytest.log
HM_DEBUG_TIMING=1 timeout 900 python bench.py > $O/${T}_bench.json 2> $O/${T}_bench.err; echo "bench $?"
tail -c 300 $O/${T}_bench.json
for v in "HM_EVAL_SPLIT=0"; do
  env $v timeout 300 python bench.py --no-factor --no-cpu-baseline --steps 2 --warmup 2 > $O/${T}_bench_${v%%=*}.json 2>&1; echo "$v $?"
done
timeout 600 python scripts/ncu_step.py save /tmp/cfg4.npz > /dev/null 2>&1
HM_NCU_NOWARM=1 timeout 420 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file $O/${T}_launches.csv python scripts/ncu_step.py load /tmp/cfg4.npz > $O/${T}_ncu_list.log 2>&1
echo "ncu list $?"
HM_NCU_NOWARM=1 timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on \
      -k regex:${KREGEX:-k_eval2} --launch-skip ${KSKIP:-2} -c 1 -o $O/${T}_${KREGEX:-k_eval2}_full \
      python scripts/ncu_step.py load /tmp/cfg4.npz > $O/${T}_ncu_full.log 2>&1
echo "ncu full $?"
