#!/bin/bash
# Round-2: tiny kernels v3 (A in registers), poll backoff sweep, multi-RHS ncu.
set -u
O=gpurun_out/r2d
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_tiny.py tests/test_gpu_multi_rhs.py -q --timeout 600 -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
tail -3 $O/pytest.log
KS_TINY_TRACE=100 KS_TINY_TRACE_OUT=$O/trace_c1.txt timeout 300 python tools/run_configs.py C1 > $O/c1_trace.jsonl 2>&1; echo "trace rc=$?"
for bo in 0 20 50 100 200; do KS_TINY_BACKOFF=$bo timeout 300 python tools/run_configs.py C1 C1bs > $O/c1_bo$bo.jsonl 2> $O/c1_bo$bo.err; echo "c1 bo=$bo rc=$?"; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cgm --launch-skip 3 -c 1 -o $O/cgm8 python tools/multi_rhs_bench.py --iters 4 > $O/ncu_cgm.log 2>&1; echo "ncu rc=$?"
