#!/bin/bash
# Round-2: tiny kernels v2 (transpose warp reduction, one-barrier block sums), multi-RHS x0 fix.
set -u
O=gpurun_out/r2d
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_tiny.py tests/test_gpu_multi_rhs.py -q --timeout 600 -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
tail -3 $O/pytest.log
KS_TINY_TRACE=100 KS_TINY_TRACE_OUT=$O/trace_c1.txt timeout 300 python tools/run_configs.py C1 > $O/c1_trace.jsonl 2>&1; echo "trace rc=$?"
timeout 300 python tools/run_configs.py C1 C1bs > $O/c1.jsonl 2> $O/c1.err; echo "c1 rc=$?"
