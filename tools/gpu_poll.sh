set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/pytest_poll.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_poll.log
timeout 600 python tools/small_path_sweep.py 1024,4096 > gpurun_out/small_path3.log 2>&1; echo "sweep rc=$?"; grep '"f64"' gpurun_out/small_path3.log | cut -c1-200
timeout 600 python tools/run_configs.py C1 C3p C3 > gpurun_out/cfg_poll.json 2>/dev/null; cut -c1-220 gpurun_out/cfg_poll.json
timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/bench_poll.json 2>/dev/null; python -c "import json;d=json.loads(open('gpurun_out/bench_poll.json').read().strip().splitlines()[-1]);print(d['value'],d['per_method'],d['gpu_launches'],d['e2e']['value'])"
