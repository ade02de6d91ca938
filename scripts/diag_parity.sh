#!/bin/bash
# Exact per-block device-vs-oracle differences (diagnostics): dump the device
# result for several HM_DROP_REL values (one npz each, small configs only).
mkdir -p gpurun_out
for d in "$@"; do
  HM_DROP_REL=$d python scripts/dump_result.py lr 4 32 1e-4 gpurun_out/diag_lr2_drop$d.npz > gpurun_out/diag_lr2_drop$d.log 2>&1
done
