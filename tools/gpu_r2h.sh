#!/bin/bash
# Round-2 profiles (one GPU): bench launch list; ncu --set full of the persistent CG
# kernel, the multi-RHS GEMM kernel (K = 8), the tiny CG kernel; the read-only probe.
set -u
O=gpurun_out/r2h
mkdir -p $O
export CUDA_VISIBLE_DEVICES=0
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-extras"
timeout 600 $B > $O/plain_bench.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $B > $O/ncu_launches.log 2>&1; echo "launches rc=$?"
for t in persist multi8 tiny; do
  case $t in persist) K=k_cg_persist;; multi8) K=k_cgm;; tiny) K=k_cg_tiny;; esac
  timeout 600 python tools/ncu_target.py $t > $O/plain_$t.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -c 1 -o $O/full_$t python tools/ncu_target.py $t > $O/ncu_$t.log 2>&1; echo "$t rc=$?"
done
timeout 300 python tools/hbm_probe.py > $O/probe_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none -k regex:k_read -c 1 -o $O/full_probe python tools/hbm_probe.py > $O/ncu_probe.log 2>&1; echo "probe rc=$?"
