#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multi.py -q --timeout 300 > gpurun_out/multi4.log 2>&1; echo "multi rc=$?" >> gpurun_out/multi4.log; tail -3 gpurun_out/multi4.log
for P in 2 4; do
  for K in persistent multi; do
    timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 2965$P bench.py --gpus $P --kernels $K > gpurun_out/bench_p${P}_$K.json 2> gpurun_out/bench_p${P}_$K.err; echo "P=$P $K rc=$?"
    python -c "import json;d=json.loads(open('gpurun_out/bench_p${P}_$K.json').read().strip().splitlines()[-1]);print(d['value'],d['per_method']['cg_iters_per_s'],d['per_method']['bicgstab_iters_per_s'],d['roofline']['achieved'],d['clocks']['sm_mhz'])"
  done
done
CUDA_VISIBLE_DEVICES=0 timeout 400 python bench.py --no-cpu-baseline > gpurun_out/bench_p1_persistent.json 2>/dev/null; python -c "import json;d=json.loads(open('gpurun_out/bench_p1_persistent.json').read().strip().splitlines()[-1]);print('P1',d['value'],d['per_method']['cg_iters_per_s'],d['per_method']['bicgstab_iters_per_s'],d['roofline']['achieved'],d['clocks']['sm_mhz'])"
