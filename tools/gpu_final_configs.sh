set -u
mkdir -p gpurun_out
CUDA_VISIBLE_DEVICES=0 timeout 1200 python tools/run_configs.py C1 C2 C3 C3p C4 C1bicg C3bicg C1gmres C3gmres > gpurun_out/final_cfg_p1.json 2>/dev/null; echo "p1 rc=$?"
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29801 tools/run_configs.py C3 C3p C4 C5cg C5bs > gpurun_out/final_cfg_p4.json 2>/dev/null; echo "p4 rc=$?"
for f in gpurun_out/final_cfg_p1.json gpurun_out/final_cfg_p4.json; do python -c "
import json,sys
for l in open('$f'):
    if l.startswith('{'):
        d=json.loads(l); print(d['P'], d['config'], d['n'], round(d['iters_per_s'],2), round(d['frac_roofline_8TBps'],3), d['iters_to_tol'], '%.2e' % d['true_relres'])
"; done
