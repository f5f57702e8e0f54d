"""Where the per-iteration time of the persistent kernels goes at moderate n: the K1
GEMV alone (ks_time_matvec, back-to-back launches on the rank's shard) vs one
fixed-length CG / BiCGSTAB iteration (tol = 0), per rank, at P = 1, 2, 4 (single
process).  overhead = iteration - GEMVs: barriers, vector phases, exchanges.
-> gpurun_out/overhead_split.json"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1511_07174_b200 as ks
import synth
res = []
for P in [p for p in (1, 2, 4) if p <= torch.cuda.device_count()]:
    for n in (16384, 65536):
        for method, kind, g in (("cg", "spd", 1), ("bicgstab", "dd", 2)):
            with ks.Context(n, ngpus=P) as ctx:
                b = ctx.generate(kind, seed=synth.SEED, table=synth.spd_table(n, 1e4) if kind == "spd" else None, kd=16)
                ctx.set_option("true_residual", 0)
                t_gemv = min(ctx.time_matvec(10) for _ in range(3))
                K = 40 if n == 16384 else 8
                getattr(ctx, method)(b, tol=0.0, maxit=4, hist=False)
                _, _, r = getattr(ctx, method)(b, tol=0.0, maxit=K, hist=False)
                it = r.seconds_loop / r.iterations
                row = {"P": P, "n": n, "method": method, "us_per_iter": 1e6 * it, "us_gemv_k1": 1e6 * t_gemv,
                       "us_overhead": 1e6 * (it - g * t_gemv)}
                print(json.dumps(row), flush=True)
                res.append(row)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/overhead_split.json", "w"), indent=1)
