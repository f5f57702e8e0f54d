#!/bin/bash
# Round-2: tiny + multi-RHS tests, phase trace of k_cg_tiny, C1 timings, per-call overhead P = 1,
# multi-RHS throughput at n = 65536.
set -u
O=gpurun_out/r2c
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_tiny.py tests/test_gpu_multi_rhs.py tests/test_gpu_parity.py -q --timeout 600 -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
tail -3 $O/pytest.log
KS_TINY_TRACE=100 KS_TINY_TRACE_OUT=$O/trace_c1.txt timeout 300 python tools/run_configs.py C1 > $O/c1_trace.jsonl 2>&1; echo "trace rc=$?"
timeout 300 python tools/run_configs.py C1 C1bs > $O/c1.jsonl 2> $O/c1.err; echo "c1 rc=$?"
timeout 300 python tools/call_overhead.py --out $O/call_overhead_p1.json > $O/co1.log 2>&1; echo "co1 rc=$?"
timeout 600 python tools/multi_rhs_bench.py > $O/multi.jsonl 2> $O/multi.err; echo "multi rc=$?"
