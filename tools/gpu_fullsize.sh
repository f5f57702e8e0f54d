set -u
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt
timeout 1800 python -m pytest tests/test_gpu_fullsize.py -q -x --timeout 1200 -p no:cacheprovider --durations=10 > gpurun_out/pytest_fullsize.log 2>&1; echo "pytest rc=$?"; tail -16 gpurun_out/pytest_fullsize.log
