set -u
mkdir -p gpurun_out
timeout 300 python tools/ncu_target.py k1t > gpurun_out/t_k1t.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1t_gemv -s 1 -c 1 -o gpurun_out/prof_k1t python tools/ncu_target.py k1t > gpurun_out/ncu_k1t.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/ncu_k1t.log
