#!/bin/bash
T=${TAG:-r1u}
O=gpurun_out
mkdir -p $O
timeout 600 python scripts/ncu_step.py save /tmp/cfg4.npz > /dev/null 2>&1
HM_NCU_NOWARM=1 timeout 420 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file $O/${T}_launches.csv python scripts/ncu_step.py load /tmp/cfg4.npz > $O/${T}_ncu_list.log 2>&1
echo "ncu list $?"
