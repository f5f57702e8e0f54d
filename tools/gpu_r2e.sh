#!/bin/bash
# tiny exchange variants: LL (0) vs ready flags (1)
set -u
O=gpurun_out/r2e
mkdir -p $O
for xm in 0 1; do
  KS_TINY_XCHG=$xm timeout 300 python tools/run_configs.py C1 C1bs > $O/c1_x$xm.jsonl 2> $O/c1_x$xm.err; echo "c1 x=$xm rc=$?"
  KS_TINY_XCHG=$xm KS_TINY_TRACE=100 KS_TINY_TRACE_OUT=$O/trace_x$xm.txt timeout 300 python tools/run_configs.py C1 > /dev/null 2>&1
done
KS_TINY_XCHG=1 timeout 900 python -m pytest tests/test_gpu_tiny.py -q --timeout 600 -p no:cacheprovider > $O/pytest_x1.log 2>&1; echo "pytest x1 rc=$?"
