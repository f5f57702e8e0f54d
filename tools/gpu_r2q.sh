#!/bin/bash
set -u
O=gpurun_out/r2q
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_multi_rhs.py tests/test_gpu_tiny.py -q --timeout 600 -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -2 $O/pytest.log
CUDA_VISIBLE_DEVICES=0 timeout 900 python tools/multi_rhs_bench.py --iters 10 --method bicgstab > $O/multi_bs.jsonl 2> $O/multi_bs.err; echo "mbs rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29612 tools/run_configs.py C16cg C16bs > $O/configs_p4.jsonl 2> $O/configs_p4.err; echo "cfg4 rc=$?"
