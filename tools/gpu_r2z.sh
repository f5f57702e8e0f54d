#!/bin/bash
# ncu --set full of the current tiny kernels (C1: k_cg_tiny, k_bs_tiny on ceil(m/8) CTAs)
set -u
O=gpurun_out/r2z
mkdir -p $O
for t in tiny tinybs; do
  k=$([ $t = tiny ] && echo k_cg_tiny || echo k_bs_tiny)
  timeout 300 python tools/ncu_target.py $t > $O/t_$t.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o $O/prof_$t python tools/ncu_target.py $t > $O/ncu_$t.log 2>&1; echo "ncu $t rc=$?"; tail -2 $O/ncu_$t.log
done
