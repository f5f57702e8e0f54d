set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_multi.py tests/test_gpu_parity.py -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_e2e4.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_e2e4.log
for P in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 2966$P bench.py --gpus $P > gpurun_out/bench_e2e_p$P.json 2> gpurun_out/bench_e2e_p$P.err; echo "bench p$P rc=$?"
  python -c "import json;d=json.loads(open('gpurun_out/bench_e2e_p$P.json').read().strip().splitlines()[-1]);print($P, d['value'], d['e2e']['value'], d['e2e_solve']['value'], d['env'])"
done
