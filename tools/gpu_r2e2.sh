#!/bin/bash
# emulated ranks on one GPU (one cooperative launch for all ranks' tiny kernels) + shared/race/tiny tests
set -u
O=gpurun_out/r2e2
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 --tb=short -p no:cacheprovider -k "shared or race or tiny" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -15 $O/pytest.log
