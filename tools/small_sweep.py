"""C1-class latency: persistent grid size x GEMV shape at small n (1 GPU)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1511_07174_b200 as ks
import synth
res = []
for n in (1024, 4096):
    for method, kind in (("cg", "spd"), ("bicgstab", "dd")):
        with ks.Context(n) as ctx:
            b = ctx.generate(kind, seed=synth.SEED, table=synth.spd_table(n, 1e3) if kind == "spd" else None, kd=16)
            ctx.set_option("true_residual", 0)
            for rows, unroll in ((0, 0), (4, 2)):
                for grid in (32, 64, 148, 296, 0):
                    ctx.set_option("gemv_rows", rows); ctx.set_option("gemv_unroll", unroll)
                    ctx.set_option("persist_grid", grid)
                    getattr(ctx, method)(b, tol=0.0, maxit=64, hist=False)
                    K = 640
                    _, _, r = getattr(ctx, method)(b, tol=0.0, maxit=K, hist=False)
                    _, _, r2 = getattr(ctx, method)(b, tol=1e-10)
                    row = {"n": n, "method": method, "rows": rows or 2, "grid": grid,
                           "us_per_iter": 1e6 * r.seconds_loop / K, "solve_ms": 1e3 * r2.seconds_total,
                           "iters": r2.iterations}
                    print(json.dumps(row), flush=True); res.append(row)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/small_sweep.json", "w"), indent=1)
