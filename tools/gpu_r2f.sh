#!/bin/bash
# Round-2 4-GPU validation after the one-launch start/end, fused x gather, rendezvous,
# tiny and multi-RHS kernels: every GPU test, bench P = 4 (self-launch) and P = 1,
# per-call overhead P = 1 / 4, exchange cost.
set -u
O=gpurun_out/r2f
mkdir -p $O
nvidia-smi --query-gpu=index,name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -rs > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
tail -3 $O/pytest.log
timeout 600 python bench.py --gpus 4 --steps 20 --warmup 5 > $O/bench4.json 2> $O/bench4.err; echo "bench4 rc=$?"
timeout 600 python bench.py --gpus 2 --steps 20 --warmup 5 > $O/bench2.json 2> $O/bench2.err; echo "bench2 rc=$?"
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench1.json 2> $O/bench1.err; echo "bench1 rc=$?"
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29611 tools/call_overhead.py --out $O/call_overhead_p4.json > $O/co4.log 2>&1; echo "co4 rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29612 tools/run_configs.py C16cg C16bs C3 C3p > $O/configs_p4.jsonl 2> $O/configs_p4.err; echo "cfg4 rc=$?"
CUDA_VISIBLE_DEVICES=0 timeout 600 python tools/run_configs.py C16cg C16bs > $O/configs_p1.jsonl 2> $O/configs_p1.err; echo "cfg1 rc=$?"
