set -u
mkdir -p gpurun_out
CMD="python bench.py --steps 16 --warmup 3 --no-cpu-baseline"
export CUDA_VISIBLE_DEVICES=0
timeout 300 $CMD > gpurun_out/plain_p.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-k_cg_persist} -s 1 -c 1 -o gpurun_out/prof_${KNAME:-persist2} $CMD > gpurun_out/ncu_persist2.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/ncu_persist2.log
