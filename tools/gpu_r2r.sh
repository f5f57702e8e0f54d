#!/bin/bash
# Full 4-GPU validation of the round-2 state: every GPU test, bench P = 1/2/4 (self-launch),
# C3/C3'/C4 at P = 4, soak.
set -u
O=gpurun_out/r2r
mkdir -p $O
nvidia-smi --query-gpu=index,name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt
timeout 2700 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -rs > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -3 $O/pytest.log
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench1.json 2> $O/bench1.err; echo "bench1 rc=$?"
timeout 600 python bench.py --gpus 2 --steps 20 --warmup 5 > $O/bench2.json 2> $O/bench2.err; echo "bench2 rc=$?"
timeout 600 python bench.py --gpus 4 --steps 20 --warmup 5 > $O/bench4.json 2> $O/bench4.err; echo "bench4 rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29612 tools/run_configs.py C3 C3p C4 C16cg C16bs > $O/configs_p4.jsonl 2> $O/configs_p4.err; echo "cfg4 rc=$?"
timeout 900 python tools/soak.py 4 300 > $O/soak_p4.json 2> $O/soak_p4.err; echo "soak4 rc=$?"; tail -c 300 $O/soak_p4.json
