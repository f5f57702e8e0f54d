#!/bin/bash
# Round-2: tiny kernels + one-launch start/end: parity tests, C1 latency tiny vs small,
# per-call overhead at P = 1, ncu of the steady-state k_cg_tiny launch.
set -u
O=gpurun_out/r2b
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_tiny.py tests/test_gpu_parity.py tests/test_gpu_bench.py -q --timeout 600 -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
tail -3 $O/pytest.log
for t in 1 0; do KS_TINY=$t timeout 300 python tools/run_configs.py C1 C1bs > $O/c1_tiny$t.jsonl 2> $O/c1_tiny$t.err; echo "c1 tiny=$t rc=$?"; done
timeout 300 python tools/call_overhead.py --out $O/call_overhead_p1.json > $O/co1.log 2>&1; echo "co1 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_cg_tiny --launch-skip 1 -c 1 -o $O/cg_tiny python tools/run_configs.py C1 > $O/ncu_cg.log 2>&1; echo "ncu rc=$?"
