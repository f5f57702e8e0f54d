set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_multi.py -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_sp.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_sp.log
timeout 600 python tools/exchange_cost.py > gpurun_out/xc4.log 2>&1; echo "xc rc=$?"; grep '"fused": 1' gpurun_out/xc4.log
timeout 900 python tools/soak.py 4 1000 2>/dev/null | tail -1
