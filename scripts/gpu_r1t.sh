#!/bin/bash
T=${TAG:-r1t}
O=gpurun_out
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${T}_smoke.log 2>&1; echo "smoke $?"; tail -1 $O/${T}_smoke.log
timeout 900 python -m pytest tests -m gpu -x -q > $O/${T}_pytest.log 2>&1; echo "pytest $?"; tail -2 $O/${T}_pytest.log
HM_DEBUG_TIMING=1 timeout 900 python bench.py > $O/${T}_bench.json 2> $O/${T}_bench.err; echo "bench $?"
tail -c 300 $O/${T}_bench.json
