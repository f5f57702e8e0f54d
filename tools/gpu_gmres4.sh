#!/bin/bash
# Fused persistent GMRES at P = 2/4: multi-GPU tests, GMRES(30) configs both modes, small-n grid sweep.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_parity.py -q -x --timeout 300 -p no:cacheprovider -k "gmres or multi or small" > gpurun_out/gmres4.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/gmres4.log
for P in 2 4; do
  for MODE in 1 0; do
    KS_PERSISTENT=$MODE timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 2975$P tools/run_configs.py C3gmres C1gmres > gpurun_out/gmres_p${P}_m$MODE.json 2> gpurun_out/gmres_p${P}_m$MODE.err; echo "P=$P persistent=$MODE rc=$?"; cat gpurun_out/gmres_p${P}_m$MODE.json
  done
done
CUDA_VISIBLE_DEVICES=0 timeout 300 python tools/small_grid_sweep.py > gpurun_out/small_grid.log 2>&1; echo "grid sweep rc=$?"; cat gpurun_out/small_grid.log
