#!/bin/bash
# emulated ranks on one GPU: persistent + tiny kernels of all ranks in one cooperative launch
set -u
O=gpurun_out/r2e3
mkdir -p $O
timeout 2000 python -m pytest tests -m gpu -q --timeout 600 --tb=short -p no:cacheprovider -k "shared or emulated or race or tiny" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -25 $O/pytest.log
