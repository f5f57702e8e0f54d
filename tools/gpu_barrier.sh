set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/pytest_parity.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_parity.log
timeout 600 python tools/small_path_sweep.py 1024,2048,4096 > gpurun_out/small_path2.log 2>&1; echo "sweep rc=$?"; grep '"f64"' gpurun_out/small_path2.log
timeout 600 python tools/run_configs.py C1 C1gmres C3p > gpurun_out/cfg_barrier.json 2>/dev/null; cat gpurun_out/cfg_barrier.json | cut -c1-300
