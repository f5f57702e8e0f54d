#!/bin/bash
set -u
O=gpurun_out/r2j
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_multi_rhs.py -q --timeout 600 -p no:cacheprovider > $O/pytest_mrhs.log 2>&1; echo "pytest mrhs rc=$?" >> $O/pytest_mrhs.log; tail -2 $O/pytest_mrhs.log
timeout 900 python tools/multi_rhs_bench.py > $O/multi_p1.jsonl 2> $O/multi_p1.err; echo "multi p1 rc=$?"
