#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu4.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu4.log
tail -4 gpurun_out/pytest_gpu4.log
CUDA_VISIBLE_DEVICES=0 timeout 300 python tools/hbm_probe.py 32 > gpurun_out/hbm_probe.log 2>&1; tail -8 gpurun_out/hbm_probe.log
CUDA_VISIBLE_DEVICES=0 timeout 300 python tools/small_n.py > gpurun_out/small_n.log 2>&1; cat gpurun_out/small_n.log | tail -20
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29614 bench.py --gpus 4 > gpurun_out/bench_p4.json 2> gpurun_out/bench_p4.err; echo "bench4 rc=$?"; cat gpurun_out/bench_p4.json
