#!/bin/bash
set -u
O=gpurun_out/r2k
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_multi_rhs.py tests/test_gpu_tiny.py -q --timeout 600 -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -2 $O/pytest.log
timeout 900 python tools/tiny_xchg.py > $O/tiny_xchg.jsonl 2> $O/tiny_xchg.err; echo "xchg rc=$?"
CUDA_VISIBLE_DEVICES=0 timeout 900 python tools/multi_rhs_bench.py > $O/multi_p1.jsonl 2> $O/multi_p1.err; echo "multi p1 rc=$?"
timeout 1500 python -m pytest tests/test_gpu_multi.py -q --timeout 900 -p no:cacheprovider -k "small or torchrun or edge or partial or rendezvous" > $O/pytest_multi.log 2>&1; echo "pytest multi rc=$?" >> $O/pytest_multi.log; tail -2 $O/pytest_multi.log
