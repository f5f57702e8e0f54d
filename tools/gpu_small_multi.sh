set -u
mkdir -p gpurun_out
CUDA_VISIBLE_DEVICES=0 timeout 600 python tools/run_configs.py C2 C2bs C16cg C16bs > gpurun_out/sm_p1.json 2>/dev/null
for P in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 2995$P tools/run_configs.py C2 C2bs C16cg C16bs > gpurun_out/sm_p$P.json 2>/dev/null; echo "P=$P rc=$?"
done
for P in 1 2 4; do python -c "
import json
for l in open('gpurun_out/sm_p$P.json'):
    if l.startswith('{'):
        d=json.loads(l); print($P, d['config'], d['n'], round(d['iters_per_s'],1), round(d['frac_roofline_8TBps'],3))
"; done
