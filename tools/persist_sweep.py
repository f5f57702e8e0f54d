"""Persistent-kernel GEMV tile shapes at n = 65536 (1 GPU): iterations/s and the
per-GEMV streaming rate, repeated to show the run-to-run spread."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1511_07174_b200 as ks
import synth
n = 65536
res = []
for method, kind in (("cg", "spd"), ("bicgstab", "dd")):
    with ks.Context(n) as ctx:
        b = ctx.generate(kind, seed=synth.SEED, table=synth.spd_table(n, 1e4) if kind == "spd" else None, kd=16)
        ctx.set_option("true_residual", 0); ctx.set_option("profile_gemv", 1)
        K = 32 if method == "cg" else 16
        for rep in range(2):
            for rows, unroll in ((0, 0), (4, 4), (2, 4)):
                ctx.set_option("gemv_rows", rows); ctx.set_option("gemv_unroll", unroll)
                getattr(ctx, method)(b, tol=0.0, maxit=4, hist=False)
                _, _, r = getattr(ctx, method)(b, tol=0.0, maxit=K, hist=False)
                row = {"method": method, "rows": rows or 4, "unroll": unroll or 2, "rep": rep,
                       "iters_per_s": K / r.seconds_loop,
                       "GBps_per_gemv": 8.0 * n * n * r.gemv_launches / r.seconds_gemv / 1e9}
                print(json.dumps(row), flush=True); res.append(row)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/persist_sweep.json", "w"), indent=1)
