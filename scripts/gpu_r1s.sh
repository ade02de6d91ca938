#!/bin/bash
# final-state check: smoke, parity, bench, ncu launch list, full capture of the dominant kernel
T=${TAG:-r1s}
O=gpurun_out
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${T}_smoke.log 2>&1; echo "smoke $?"; tail -1 $O/${T}_smoke.log
timeout 900 python -m pytest tests -m gpu -x -q > $O/${T}_pytest.log 2>&1; echo "pytest $?"; tail -2 $O/${T}_pytest.log
HM_DEBUG_TIMING=1 timeout 900 python bench.py > $O/${T}_bench.json 2> $O/${T}_bench.err; echo "bench $?"
tail -c 300 $O/${T}_bench.json
timeout 300 python bench.py --impl reference --steps 1 --warmup 0 > $O/${T}_bench_ref.json 2>&1; echo "ref $?"
timeout 600 python scripts/ncu_step.py save /tmp/cfg4.npz > /dev/null 2>&1
HM_NCU_NOWARM=1 timeout 420 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file $O/${T}_launches.csv python scripts/ncu_step.py load /tmp/cfg4.npz > $O/${T}_ncu_list.log 2>&1
echo "ncu list $?"
HM_NCU_NOWARM=1 timeout 480 ncu --profile-from-start off --set full --clock-control none --import-source on \
      -k regex:k_qr_blocked --launch-skip 2 -c 1 -o $O/${T}_k_qr_blocked_full \
      python scripts/ncu_step.py load /tmp/cfg4.npz > $O/${T}_ncu_full.log 2>&1
echo "ncu full $?"
