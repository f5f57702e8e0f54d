#!/bin/bash
# Round-2 final multi-GPU validation (gpurun --gpus 4): every GPU test (P = 2 / 4 GPU
# layouts, race tests, shared layouts), bench self-launch P = 2 / 4, soak.
set -u
O=gpurun_out/r2y
mkdir -p $O
nvidia-smi --query-gpu=index,name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt
timeout 2700 python -m pytest tests -m gpu -q --timeout 900 --tb=short -p no:cacheprovider > $O/pytest_gpu4.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu4.log
tail -5 $O/pytest_gpu4.log
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py > $O/bench_p1.json 2> $O/bench_p1.err; echo "bench p1 rc=$?"
python -c "import json;d=json.loads(open('$O/bench_p1.json').read().strip().splitlines()[-1]);print(1, d['value'], d['e2e']['value'], d['roofline']['frac'], d['clocks'], json.dumps(d.get('extras', {}).get('c1_latency')))"
for P in 2 4; do
  timeout 600 python bench.py --gpus $P > $O/bench_p$P.json 2> $O/bench_p$P.err; echo "bench p$P rc=$?"
  python -c "import json;d=json.loads(open('$O/bench_p$P.json').read().strip().splitlines()[-1]);print($P, d['n_gpus'], d['value'], d['e2e']['value'], d['roofline']['frac'], d['clocks'])"
done
timeout 600 python tools/soak.py 4 200 > $O/soak_p4.json 2> $O/soak_p4.err; echo "soak4 rc=$?"; tail -c 300 $O/soak_p4.json
timeout 900 python tools/ll_ab.py > $O/ll_ab.jsonl 2> $O/ll_ab.err; echo "ll_ab rc=$?"; cat $O/ll_ab.jsonl
