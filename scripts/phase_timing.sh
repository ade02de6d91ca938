#!/bin/bash
# Rebuild libhm with -DHM_PHASE_TIMING (per-phase cycle printf of CTA 0 in the
# TRUNC kernels) and run single-stack TRUNCs at the given shapes.  Diagnostics only.
set -e
cd "$(dirname "$0")/../paper_1703_09085_b200"
for o in svd qr qr_reg; do make -B NVFLAGS="-gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -lineinfo -Xcompiler -fPIC,-ffp-contract=off -DHM_PHASE_TIMING" build/$o.o > /dev/null 2>&1; done
make > /dev/null 2>&1
cd ..
for s in "$@"; do
  echo "== $s"
  python scripts/one_trunc.py $s 2>&1 | tail -24
done
