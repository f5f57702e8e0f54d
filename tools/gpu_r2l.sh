#!/bin/bash
set -u
O=gpurun_out/r2l
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_tiny.py tests/test_gpu_multi_rhs.py -q --timeout 600 -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -2 $O/pytest.log
timeout 1500 python -m pytest tests/test_gpu_multi.py -q --timeout 900 -p no:cacheprovider -k "small or edge" > $O/pytest_multi.log 2>&1; echo "pytest multi rc=$?" >> $O/pytest_multi.log; tail -2 $O/pytest_multi.log
CUDA_VISIBLE_DEVICES=0 timeout 300 python tools/run_configs.py C1 C1bs > $O/c1.jsonl 2> $O/c1.err; echo "c1 rc=$?"
timeout 900 python tools/soak.py 4 400 > $O/soak_p4.json 2> $O/soak_p4.err; echo "soak4 rc=$?"; tail -c 600 $O/soak_p4.json
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29621 tools/soak.py 4 300 > $O/soak_tr4.json 2> $O/soak_tr4.err; echo "soaktr rc=$?"; tail -c 600 $O/soak_tr4.json
timeout 600 python tools/soak.py 1 300 > $O/soak_p1.json 2> $O/soak_p1.err; echo "soak1 rc=$?"; tail -c 400 $O/soak_p1.json
