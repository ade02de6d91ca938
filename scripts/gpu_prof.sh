#!/bin/bash
# ncu evidence for one bench step of config 4 (one gpurun call = one ncu use):
# launch list with DRAM bytes (-> profiles/<tag>_traffic.json) and full
# captures of the top kernels.  Usage: bash scripts/gpu_prof.sh TAG
TAG=${1:-r2}
OUT=gpurun_out
mkdir -p $OUT
python scripts/ncu_step.py save /tmp/cfg4.npz > $OUT/${TAG}_save.log 2>&1 &&
python scripts/ncu_step.py load /tmp/cfg4.npz > $OUT/${TAG}_plain.log 2>&1 &&
timeout 1500 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file $OUT/${TAG}_launches.csv python scripts/ncu_step.py load /tmp/cfg4.npz \
    > $OUT/${TAG}_ncu_list.log 2>&1
echo "launch list exit $?"
python scripts/ncu_traffic.py $OUT/${TAG}_launches.csv $OUT/${TAG}_traffic.json > $OUT/${TAG}_traffic.txt 2>&1
head -25 $OUT/${TAG}_traffic.txt
# full captures: the 768- and 1536-row QR instantiations, the SVD, the fused TRUNC, the eval
for spec in "k_qr_blocked<256, 2, 4, false>:2" "k_qr_blocked<512, 1, 4, false>:2" "k_svd:6" "k_trunc_small:6" "k_eval2:6"; do
  name=${spec%:*}; skip=${spec##*:}
  safe=$(echo "$name" | tr -c 'a-zA-Z0-9_\n' '_')
  timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
      -k "regex:^$(echo "$name" | sed 's/[<>, ]/./g')" --launch-skip $skip -c 1 -o $OUT/${TAG}_${safe} \
      python scripts/ncu_step.py load /tmp/cfg4.npz > $OUT/${TAG}_${safe}.log 2>&1
  echo "full $name exit $?"
done
