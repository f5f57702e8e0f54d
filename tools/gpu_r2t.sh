#!/bin/bash
# shared-device layouts (P ranks on GPU 0) on a 1-GPU box
set -u
O=gpurun_out/r2t
mkdir -p $O
nvidia-smi -L > $O/gpus.txt
timeout 300 python -m pytest tests/test_gpu_multi.py -q -x --timeout 120 -p no:cacheprovider -k "shared2 and gemv_and_cg" > $O/first.log 2>&1; echo "first rc=$?" >> $O/first.log; tail -3 $O/first.log
timeout 2400 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -k shared > $O/pytest_shared.log 2>&1; echo "pytest rc=$?" >> $O/pytest_shared.log; tail -15 $O/pytest_shared.log
