#!/bin/bash
set -u
O=gpurun_out/r2p
mkdir -p $O
timeout 1200 python tools/overhead_split.py > $O/overhead_split.jsonl 2> $O/overhead_split.err; echo "split rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29612 tools/run_configs.py C16cg C16bs > $O/configs_p4.jsonl 2> $O/configs_p4.err; echo "cfg4 rc=$?"
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench1.json 2> $O/bench1.err; echo "bench1 rc=$?"
for sh in 0 1 2; do CUDA_VISIBLE_DEVICES=0 KS_MULTI_SHAPE=$sh timeout 900 python tools/multi_rhs_bench.py --iters 10 > $O/multi_shape$sh.jsonl 2> $O/multi_shape$sh.err; echo "shape $sh rc=$?"; done
timeout 1500 python -m pytest tests/test_gpu_multi_rhs.py tests/test_gpu_parity.py -q --timeout 900 -p no:cacheprovider -x -k "multi_rhs or persistent or large_shard or cg_parity or bicgstab_parity" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -2 $O/pytest.log
