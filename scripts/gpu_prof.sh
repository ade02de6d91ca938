#!/bin/bash
# ncu evidence for one hm_addmul step (one gpurun call = one ncu use): launch
# list with DRAM bytes (-> <tag>_traffic.json) and full captures of the top
# kernels.  NCU_L (default 5): icosphere level of the profiled product (see
# scripts/ncu_step.py).  Usage: bash scripts/gpu_prof.sh TAG
TAG=${1:-r2}
export NCU_L=${NCU_L:-5}
OUT=gpurun_out
mkdir -p $OUT
python scripts/ncu_step.py save /tmp/cfgL.npz > $OUT/${TAG}_save.log 2>&1 &&
python scripts/ncu_step.py load /tmp/cfgL.npz > $OUT/${TAG}_plain.log 2>&1 &&
timeout 1200 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file $OUT/${TAG}_launches.csv python scripts/ncu_step.py load /tmp/cfgL.npz \
    > $OUT/${TAG}_ncu_list.log 2>&1
echo "launch list exit $?"
python scripts/ncu_traffic.py $OUT/${TAG}_launches.csv $OUT/${TAG}_traffic.json > $OUT/${TAG}_traffic.txt 2>&1
head -25 $OUT/${TAG}_traffic.txt
python scripts/ncu_pick.py $OUT/${TAG}_launches.csv > $OUT/${TAG}_specs.txt
cat $OUT/${TAG}_specs.txt
while IFS=: read -r rx name skip; do
  [ -z "$rx" ] && continue
  timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on \
      --kernel-name-base mangled -k "regex:$rx" --launch-skip $skip -c 1 -o $OUT/${TAG}_${name} \
      python scripts/ncu_step.py load /tmp/cfgL.npz > $OUT/${TAG}_${name}.log 2>&1
  echo "full $name exit $?"
  # gpurun_out is limited to 64 MiB: keep the CSV exports, not the reports
  if [ -f $OUT/${TAG}_${name}.ncu-rep ]; then
    ncu -i $OUT/${TAG}_${name}.ncu-rep --page details --csv > $OUT/${TAG}_k_${name}_full_details.csv 2>/dev/null
    python scripts/ncu_src.py $OUT/${TAG}_${name}.ncu-rep 25 > $OUT/${TAG}_k_${name}_source_summary.txt 2>/dev/null
    rm -f $OUT/${TAG}_${name}.ncu-rep
  fi
done < $OUT/${TAG}_specs.txt
