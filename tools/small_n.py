"""Latency-bound small-n path (C1): microseconds per iteration, graphs on/off."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1511_07174_b200 as ks
import synth
res = []
for n in (1024, 4096, 16384):
    with ks.Context(n) as ctx:
        b = ctx.generate("spd", seed=synth.SEED, table=synth.spd_table(n, 1e3))
        bd = ctx.generate("dd", seed=synth.SEED, kd=16) if False else None
        for graphs in (0, 1):
            for batch in (16, 64):
                ctx.set_option("use_graphs", graphs); ctx.set_option("poll_batch", batch)
                ctx.set_option("true_residual", 0)
                ctx.cg(b, tol=0.0, maxit=200)
                x, h, r = ctx.cg(b, tol=0.0, maxit=1000)
                x2, h2, r2 = ctx.cg(b, tol=1e-10)
                row = {"n": n, "method": "cg", "graphs": graphs, "batch": batch,
                       "us_per_iter": 1e6 * r.seconds_loop / r.iterations,
                       "solve_ms_to_tol": 1e3 * r2.seconds_total, "iters_to_tol": r2.iterations}
                print(json.dumps(row), flush=True); res.append(row)
    with ks.Context(n) as ctx:
        b = ctx.generate("dd", seed=synth.SEED, kd=16)
        for graphs in (0, 1):
            ctx.set_option("use_graphs", graphs); ctx.set_option("poll_batch", 16); ctx.set_option("true_residual", 0)
            ctx.bicgstab(b, tol=0.0, maxit=100)
            x, h, r = ctx.bicgstab(b, tol=0.0, maxit=500)
            row = {"n": n, "method": "bicgstab", "graphs": graphs, "batch": 16,
                   "us_per_iter": 1e6 * r.seconds_loop / r.iterations}
            print(json.dumps(row), flush=True); res.append(row)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/small_n.json", "w"), indent=1)
