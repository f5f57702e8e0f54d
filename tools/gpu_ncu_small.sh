set -u
mkdir -p gpurun_out
timeout 300 python tools/ncu_target.py small > gpurun_out/t_small.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cg_small -s 1 -c 1 -o gpurun_out/prof_small python tools/ncu_target.py small > gpurun_out/ncu_small.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/ncu_small.log
