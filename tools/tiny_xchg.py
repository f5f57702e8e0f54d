"""Per-iteration cost at small n on P = 1, 2, 4 GPUs (single-process mode): the tiny
kernels (LL exchange; P > 1 over NVLink) vs the round-1 small-n / general kernels
(tiny = 0).  us/iteration -> gpurun_out/tiny_xchg.json"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1511_07174_b200 as ks
import synth
res = []
for P in [p for p in (1, 2, 4, 8) if p <= torch.cuda.device_count()]:
    for n in (512, 1024):
        for method, kind in (("cg", "spd"), ("bicgstab", "dd")):
            with ks.Context(n, ngpus=P) as ctx:
                b = ctx.generate(kind, seed=synth.SEED, table=synth.spd_table(n, 1e3) if kind == "spd" else None, kd=16)
                ctx.set_option("true_residual", 0)
                for tiny in (1, 0):
                    ctx.set_option("tiny", tiny)
                    K = 120 if method == "cg" else 30
                    getattr(ctx, method)(b, tol=0.0, maxit=8, hist=False)
                    _, _, r = getattr(ctx, method)(b, tol=0.0, maxit=K, hist=False)
                    row = {"P": P, "n": n, "method": method, "tiny": tiny, "iters": r.iterations,
                           "us_per_iter": 1e6 * r.seconds_loop / max(1, r.iterations)}
                    print(json.dumps(row), flush=True)
                    res.append(row)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/tiny_xchg.json", "w"), indent=1)
