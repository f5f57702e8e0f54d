#!/bin/bash
set -u
O=gpurun_out/r2o
mkdir -p $O
timeout 1200 python tools/overhead_split.py > $O/overhead_split.jsonl 2> $O/overhead_split.err; echo "split rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29631 tools/multi_rhs_bench.py --iters 10 > $O/multi_p4.jsonl 2> $O/multi_p4.err; echo "multi p4 rc=$?"
export CUDA_VISIBLE_DEVICES=0
timeout 600 python tools/ncu_target.py multi8 > $O/plain_multi8.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cgm -c 1 -o $O/full_multi8 python tools/ncu_target.py multi8 > $O/ncu_multi8.log 2>&1; echo "ncu rc=$?"
