#!/bin/bash
# shared-device diagnosis: per-case subprocesses, then the failing tests with tracebacks
set -u
O=gpurun_out/r2v
mkdir -p $O
timeout 1500 python tools/shared_diag.py > $O/diag.jsonl 2> $O/diag.err; echo "diag rc=$?"; cat $O/diag.jsonl
for k in "multi_bicgstab and shared2" "edge_cases and shared2" "gmres and 0-shared2" "persistent_fused and shared4" "gemv_and_cg and shared4"; do
  timeout 400 python -m pytest tests/test_gpu_multi.py -x -q --timeout 180 --tb=short -p no:cacheprovider -k "$k" >> $O/tests.log 2>&1; echo "[$k] rc=$?" >> $O/tests.log
done
grep -E "rc=|Error|error|assert|KsError" $O/tests.log | head -60
