#!/bin/bash
# Does ncu follow the library?  Plain run, then a short launch list (first 60
# launches of the profiled step) with the private pool and with HM_POOL=default.
OUT=gpurun_out; mkdir -p $OUT
python scripts/ncu_step.py save /tmp/cfg4.npz > $OUT/np_save.log 2>&1
python scripts/ncu_step.py load /tmp/cfg4.npz > $OUT/np_plain.log 2>&1 && echo plain ok
HM_POOL=default timeout 400 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
   --log-file $OUT/np_default.csv python scripts/ncu_step.py load /tmp/cfg4.npz > $OUT/np_default.log 2>&1
echo "default pool exit $? $(wc -l < $OUT/np_default.csv)"
timeout 400 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
   --log-file $OUT/np_private.csv python scripts/ncu_step.py load /tmp/cfg4.npz > $OUT/np_private.log 2>&1
echo "private pool exit $? $(wc -l < $OUT/np_private.csv)"
