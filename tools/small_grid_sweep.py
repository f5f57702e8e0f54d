"""Small-n kernels: us/iteration vs the CTA count (KS_OPT_PERSIST_GRID caps it), C1-class n."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1511_07174_b200 as ks
import synth
res = []
for n in (1024, 2048):
    for method, kind in (("cg", "spd"), ("bicgstab", "dd")):
        with ks.Context(n) as ctx:
            b = ctx.generate(kind, seed=synth.SEED, table=synth.spd_table(n, 1e3) if kind == "spd" else None, kd=16)
            ctx.set_option("true_residual", 0)
            ctx.set_option("small", 1)
            for grid in (32, 64, 96, 128, 148, 192, 256, 0):
                ctx.set_option("persist_grid", grid)
                getattr(ctx, method)(b, tol=0.0, maxit=64, hist=False)
                _, _, r = getattr(ctx, method)(b, tol=0.0, maxit=1000 if method == "cg" else 300, hist=False)
                row = {"n": n, "method": method, "grid_cap": grid,
                       "us_per_iter": 1e6 * r.seconds_loop / max(1, r.iterations), "iters": r.iterations}
                print(json.dumps(row), flush=True)
                res.append(row)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/small_grid_sweep.json", "w"), indent=1)
