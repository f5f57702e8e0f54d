set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "persistent or small or f32 or edge or c1 or spec or strided" > gpurun_out/pytest_small.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_small.log
timeout 600 python tools/small_path_sweep.py > gpurun_out/small_path.log 2>&1; echo "sweep rc=$?"; cat gpurun_out/small_path.log | tail -45
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_e2e.json 2> gpurun_out/bench_e2e.err; echo "bench rc=$?"; cat gpurun_out/bench_e2e.json
