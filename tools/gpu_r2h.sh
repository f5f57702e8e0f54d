#!/bin/bash
# deferred row reductions in the persistent GEMV phase: A/B + parity with the switch on
set -u
O=gpurun_out/r2h
mkdir -p $O
timeout 1200 python tools/defer_ab.py > $O/defer_ab.jsonl 2> $O/defer_ab.err; echo "ab rc=$?"; cat $O/defer_ab.jsonl
KS_GEMV_DEFER=1 timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_race.py -m gpu -q --timeout 600 --tb=short -p no:cacheprovider -k "not shared" > $O/pytest_defer.log 2>&1; echo "pytest rc=$?" >> $O/pytest_defer.log; tail -4 $O/pytest_defer.log
