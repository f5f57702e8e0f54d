#!/bin/bash
# persist_shape fix (R = 1 on badly filled waves) at n = 16384 P = 1/2/4; tiny LDG.256 vs 2 x 128 A/B.
set -u
O=gpurun_out/r2i
mkdir -p $O
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29612 tools/run_configs.py C16cg C16bs > $O/configs_p4.jsonl 2> $O/configs_p4.err; echo "cfg4 rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29613 tools/run_configs.py C16cg C16bs > $O/configs_p2.jsonl 2> $O/configs_p2.err; echo "cfg2 rc=$?"
for w in 1 0 1 0; do CUDA_VISIBLE_DEVICES=0 KS_TINY_WIDE=$w timeout 300 python tools/run_configs.py C1 C1bs >> $O/c1_w$w.jsonl 2>> $O/c1.err; done; echo "c1 done"
timeout 900 python -m pytest tests/test_gpu_multi.py -q --timeout 900 -p no:cacheprovider -x -k "multi_persistent_fused or multi_bicgstab or multi_gemv_and_cg or torchrun" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -2 $O/pytest.log
