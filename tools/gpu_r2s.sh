#!/bin/bash
set -u
O=gpurun_out/r2s
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_multi_rhs.py -q --timeout 600 -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -2 $O/pytest.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29631 tools/multi_rhs_bench.py --iters 10 --method bicgstab > $O/multi_bs_p4.jsonl 2> $O/multi_bs_p4.err; echo "mbs p4 rc=$?"
timeout 900 python tools/soak.py 4 300 > $O/soak_p4.json 2> $O/soak_p4.err; echo "soak4 rc=$?"; tail -c 300 $O/soak_p4.json
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29621 tools/soak.py 4 300 > $O/soak_tr4.json 2> $O/soak_tr4.err; echo "soaktr rc=$?"; tail -c 300 $O/soak_tr4.json
