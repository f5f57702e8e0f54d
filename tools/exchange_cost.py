"""Per-iteration overhead of the fused exchange: CG / BiCGSTAB at tiny n (GEMV ~free)
on P = 1 (general persistent kernel, small-n kernels off) vs P GPUs (persistent +
fused), single-process mode.  us/iteration -> gpurun_out/exchange_cost.json"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1511_07174_b200 as ks
import synth
res = []
for P in [p for p in (1, 2, 4) if p <= torch.cuda.device_count()]:
    for n in (512, 4096):
        for method, kind in (("cg", "spd"), ("bicgstab", "dd")):
            with ks.Context(n, ngpus=P) as ctx:
                b = ctx.generate(kind, seed=synth.SEED, table=synth.spd_table(n, 1e2) if kind == "spd" else None, kd=4)
                ctx.set_option("true_residual", 0)
                ctx.set_option("small", int(os.environ.get("KS_SMALL", "0")))
                for fused in ((1, 0) if P > 1 else (1,)):
                    ctx.set_option("fused_comm", fused)
                    ctx.set_option("persistent", 2)
                    getattr(ctx, method)(b, tol=0.0, maxit=32, hist=False)
                    _, _, r = getattr(ctx, method)(b, tol=0.0, maxit=400, hist=False)
                    row = {"P": P, "n": n, "method": method, "fused": fused,
                           "persistent": ctx.get_option("persistent"), "iters": r.iterations,
                           "us_per_iter": 1e6 * r.seconds_loop / max(1, r.iterations)}
                    print(json.dumps(row), flush=True)
                    res.append(row)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/exchange_cost.json", "w"), indent=1)
