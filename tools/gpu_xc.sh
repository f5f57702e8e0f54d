set -u
mkdir -p gpurun_out
timeout 600 python tools/exchange_cost.py > gpurun_out/xc3.log 2>&1; echo "xc rc=$?"; grep '"fused": 1' gpurun_out/xc3.log
