#!/bin/bash
# final build on 2 GPUs: the tests after test_gpu_race in collection order + race + emulated
set -u
O=gpurun_out/r2f3
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_race.py tests/test_gpu_tiny.py -m gpu -q --timeout 600 --tb=short -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -8 $O/pytest.log
timeout 900 python -m pytest tests -m gpu -q --timeout 600 --tb=short -p no:cacheprovider -k "emulated or shared" > $O/pytest2.log 2>&1; echo "pytest2 rc=$?" >> $O/pytest2.log; tail -4 $O/pytest2.log
