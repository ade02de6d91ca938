#!/bin/bash
# parity tests + bench + full captures of the SVD kernels
T=${TAG:-r1g}
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/${T}_pytest.log 2>&1; echo "pytest $?"; tail -2 $O/${T}_pytest.log
HM_DEBUG_TIMING=1 timeout 900 python bench.py > $O/${T}_bench.json 2> $O/${T}_bench.err; echo "bench $?"
tail -c 300 $O/${T}_bench.json
timeout 600 python scripts/ncu_step.py save /tmp/cfg4.npz > /dev/null 2>&1
for K in k_svd k_trunc_small; do
HM_NCU_NOWARM=1 timeout 480 ncu --profile-from-start off --set full --clock-control none --import-source on \
      -k regex:$K --launch-skip 6 -c 1 -o $O/${T}_${K}_full \
      python scripts/ncu_step.py load /tmp/cfg4.npz > $O/${T}_ncu_full_$K.log 2>&1
echo "ncu full $K $?"
done
