set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_multi.py tests/test_gpu_parity.py -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_bsp.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_bsp.log
KS_SMALL=1 timeout 600 python tools/exchange_cost.py > gpurun_out/xc7.log 2>&1; echo "xc rc=$?"; grep '"fused": 1' gpurun_out/xc7.log | grep bicgstab
timeout 900 python tools/soak.py 4 3000 2>/dev/null | tail -1 | cut -c1-300
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29803 tools/soak.py 4 2000 2>/dev/null | tail -1 | cut -c1-300
KS_GUARD=1 timeout 900 python tools/guard_run.py 2>&1 | tail -2
