#!/bin/bash
set -u
O=gpurun_out/r2m
mkdir -p $O
for sh in 0 1; do CUDA_VISIBLE_DEVICES=0 KS_MULTI_SHAPE=$sh timeout 900 python tools/multi_rhs_bench.py > $O/multi_shape$sh.jsonl 2> $O/multi_shape$sh.err; echo "shape $sh rc=$?"; done
timeout 1200 python -m pytest tests/test_gpu_multi_rhs.py -q --timeout 600 -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -2 $O/pytest.log
timeout 900 python tools/soak.py 4 400 > $O/soak_p4.json 2> $O/soak_p4.err; echo "soak4 rc=$?"; tail -c 600 $O/soak_p4.json
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29621 tools/soak.py 4 300 > $O/soak_tr4.json 2> $O/soak_tr4.err; echo "soaktr rc=$?"; tail -c 600 $O/soak_tr4.json
timeout 600 python tools/soak.py 1 300 > $O/soak_p1.json 2> $O/soak_p1.err; echo "soak1 rc=$?"; tail -c 400 $O/soak_p1.json
