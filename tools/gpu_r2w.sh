#!/bin/bash
# shared4 co-residency: SM slack and hardware-queue count variants
set -u
O=gpurun_out/r2w
mkdir -p $O
for v in "KS_SHARED_SLACK=0 CUDA_DEVICE_MAX_CONNECTIONS=32" "KS_SHARED_SLACK=4" "KS_SHARED_SLACK=12" "KS_SHARED_SLACK=0"; do
  echo "== $v" >> $O/diag.jsonl
  env $v timeout 700 python tools/shared_diag.py bs1024:4 cg2048:4 cg4096:4 gm1024:2 >> $O/diag.jsonl 2>> $O/diag.err
done
cat $O/diag.jsonl
