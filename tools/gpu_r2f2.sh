#!/bin/bash
# final build on a 2-GPU box: the whole GPU suite (gpus1/gpus2/shared layouts), smoke, bench P = 1 / 2
set -u
O=gpurun_out/r2f2
mkdir -p $O
nvidia-smi --query-gpu=index,name --format=csv > $O/gpu.txt
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 --tb=short -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -6 $O/pytest.log
CUDA_VISIBLE_DEVICES=0 timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py > $O/bench_p1.json 2> $O/bench_p1.err; echo "bench p1 rc=$?"
timeout 600 python bench.py --gpus 2 > $O/bench_p2.json 2> $O/bench_p2.err; echo "bench p2 rc=$?"
for P in 1 2; do python -c "import json;d=json.loads(open('$O/bench_p$P.json').read().strip().splitlines()[-1]);print($P, d['n_gpus'], d['value'], d['e2e']['value'], d['roofline']['frac'], d['clocks'], json.dumps((d.get('extras') or {}).get('c1_latency')))"; done
