#!/bin/bash
# Round-2 first validation on a 4-GPU box: every GPU test (C3 gate at P = 1/2/4),
# bench self-launch at --gpus 4, bench P = 1, per-call overhead breakdown P = 1/4.
set -u
O=gpurun_out/r2a
mkdir -p $O
nvidia-smi --query-gpu=index,name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt
(nproc; free -g; lscpu | head -20) > $O/host.txt 2>&1
timeout 2000 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -rs > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
tail -5 $O/pytest.log
timeout 600 python bench.py --gpus 4 --steps 20 --warmup 5 > $O/bench4.json 2> $O/bench4.err; echo "bench4 rc=$?"
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench1.json 2> $O/bench1.err; echo "bench1 rc=$?"
CUDA_VISIBLE_DEVICES=0 timeout 300 python tools/call_overhead.py --out $O/call_overhead_p1.json > $O/co1.log 2>&1; echo "co1 rc=$?"
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29611 tools/call_overhead.py --out $O/call_overhead_p4.json > $O/co4.log 2>&1; echo "co4 rc=$?"
