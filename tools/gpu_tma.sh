set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "tma or persistent" > gpurun_out/pytest_tma.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_tma.log
timeout 900 python tools/persist_tma.py > gpurun_out/persist_tma.log 2>&1; echo "sweep rc=$?"; cat gpurun_out/persist_tma.log
