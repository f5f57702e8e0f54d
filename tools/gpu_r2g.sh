#!/bin/bash
# R=1 persistent tiles for badly filled waves, one-fence k_end, LDG.256 LL polls.
set -u
O=gpurun_out/r2g
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_multi.py tests/test_gpu_tiny.py -q --timeout 900 -p no:cacheprovider -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
tail -2 $O/pytest.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29612 tools/run_configs.py C16cg C16bs C3p > $O/configs_p4.jsonl 2> $O/configs_p4.err; echo "cfg4 rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29613 tools/run_configs.py C16cg C16bs > $O/configs_p2.jsonl 2> $O/configs_p2.err; echo "cfg2 rc=$?"
CUDA_VISIBLE_DEVICES=0 timeout 600 python tools/run_configs.py C16cg C16bs C1 C1bs > $O/configs_p1.jsonl 2> $O/configs_p1.err; echo "cfg1 rc=$?"
timeout 600 python bench.py --gpus 4 --steps 20 --warmup 5 > $O/bench4.json 2> $O/bench4.err; echo "bench4 rc=$?"
