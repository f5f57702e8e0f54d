#!/bin/bash
# Full validation on a 4-GPU box: all GPU tests, bench P=1/2/4, ncu (GPU 0 only).
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu4.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu4.log
tail -3 gpurun_out/pytest_gpu4.log
CUDA_VISIBLE_DEVICES=0 timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py > gpurun_out/bench_p1.json 2> gpurun_out/bench_p1.err; echo "bench p1 rc=$?"
for P in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 2967$P bench.py --gpus $P > gpurun_out/bench_p$P.json 2> gpurun_out/bench_p$P.err; echo "bench p$P rc=$?"
done
for P in 1 2 4; do python -c "import json;d=json.loads(open('gpurun_out/bench_p$P.json').read().strip().splitlines()[-1]);print($P, d['value'],d['per_method']['cg_iters_per_s'],d['per_method']['bicgstab_iters_per_s'],d['roofline']['achieved'],d['roofline']['frac'],d['clocks'])"; done
CMD="python bench.py --steps 16 --warmup 3 --no-cpu-baseline"
export CUDA_VISIBLE_DEVICES=0
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
# (one ncu per call: the --set full capture runs in its own call)
