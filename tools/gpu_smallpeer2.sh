set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_multi.py -q -x --timeout 600 -p no:cacheprovider -k "small or bicgstab or persistent or fused or torchrun" > gpurun_out/pytest_sp2.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_sp2.log
KS_SMALL=1 timeout 600 python tools/exchange_cost.py > gpurun_out/xc6.log 2>&1; echo "xc rc=$?"; grep '"fused": 1' gpurun_out/xc6.log
timeout 900 python tools/soak.py 4 1500 2>/dev/null | tail -1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29778 tools/soak.py 4 800 2>/dev/null | tail -1
