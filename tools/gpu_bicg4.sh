#!/bin/bash
# Fused BiCG (K1T + reduce-scatter in one kernel) and torchrun GMRES at P = 2/4.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x --timeout 300 -p no:cacheprovider -k "bicg or torchrun or gmres" > gpurun_out/bicg4.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/bicg4.log
for P in 2 4; do
  for F in 1 0; do
    KS_FUSED=$F timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 2985$P tools/run_configs.py C3bicg C1bicg > gpurun_out/bicg_p${P}_f$F.json 2> gpurun_out/bicg_p${P}_f$F.err; echo "P=$P fused=$F rc=$?"; cat gpurun_out/bicg_p${P}_f$F.json
  done
done
