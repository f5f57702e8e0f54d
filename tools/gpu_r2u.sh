#!/bin/bash
# Round-2 rehearsal on one GPU: shared-GPU (host-collective) layouts and race tests
# first, then the whole GPU suite, smoke, bench, ncu launch list, tiny-grid A/B.
set -u
O=gpurun_out/r2u
mkdir -p $O
nvidia-smi --query-gpu=name,driver_version,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 --tb=short -p no:cacheprovider -k "shared or race" > $O/shared_race.log 2>&1; echo "shared+race rc=$?" >> $O/shared_race.log; tail -4 $O/shared_race.log
timeout 2400 python -m pytest tests -m gpu -q --timeout 600 --tb=short -p no:cacheprovider -k "not shared and not race" > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log; tail -3 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; cat $O/bench.json
CMD="python bench.py --steps 16 --warmup 3 --no-cpu-baseline --no-extras"
timeout 300 $CMD > $O/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $CMD > $O/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
timeout 600 python tools/tiny_grid_ab.py > $O/tiny_grid_ab.jsonl 2> $O/tiny_grid_ab.err; echo "tiny grid rc=$?"; cat $O/tiny_grid_ab.jsonl
for rep in 1 2; do for occ in 4 5; do
  KS_PERSIST_OCC=$occ timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-extras > $O/occ$occ.json 2>/dev/null
  python -c "import json,sys; d=json.loads(open('$O/occ$occ.json').read().strip().splitlines()[-1]); print(json.dumps({'occ': $occ, 'rep': $rep, 'value': d['value'], 'frac': d['roofline']['frac'], 'e2e': d['e2e']['value']}))" >> $O/occ_ab.jsonl
done; done
cat $O/occ_ab.jsonl
