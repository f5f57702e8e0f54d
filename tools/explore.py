"""Quick GPU exploration: K1 timing per variant/tile, solver it/s at n=65536."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1511_07174_b200 as ks
import synth

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
out = {"n": n}
with ks.Context(n) as ctx:
    t = time.time(); b = ctx.generate("dd", seed=synth.SEED, kd=16); out["gen_dd_s"] = time.time() - t
    res = {}
    for var in (1,):   # the round-1 TMA variant (2) was removed
        for rows in (4, 8, 16):
            ctx.set_option("gemv_kernel", var); ctx.set_option("gemv_rows", rows)
            s = ctx.time_matvec(10)
            res[f"v{var}_r{rows}"] = {"ms": s * 1e3, "GBps": 8.0 * n * n / s / 1e9}
            print(var, rows, res[f"v{var}_r{rows}"], flush=True)
    out["gemv"] = res
    best = min(res, key=lambda k: res[k]["ms"])
    ctx.set_option("gemv_kernel", int(best[1])); ctx.set_option("gemv_rows", int(best.split("r")[1]))
    ctx.set_option("profile_gemv", 1)
    x, h, r = ctx.bicgstab(b, tol=1e-10)
    out["bicgstab"] = {"iters": r.iterations, "half": r.half_step_exit, "true_relres": r.true_relres,
                       "hist0": h[:3].tolist(), "ips": r.iterations / r.seconds_loop,
                       "loop_s": r.seconds_loop, "gemv_s": r.seconds_gemv, "launches": r.kernel_launches}
    print(out["bicgstab"], flush=True)
    x, h, r = ctx.bicgstab(b, tol=0.0, maxit=20)
    out["bicgstab_fixed20"] = {"ips": r.iterations / r.seconds_loop, "gemv_frac": r.seconds_gemv / r.seconds_loop}
    print(out["bicgstab_fixed20"], flush=True)
with ks.Context(n) as ctx:
    c = synth.spd_table(n, 1e4)
    b = ctx.generate("spd", seed=synth.SEED, table=c)
    ctx.set_option("gemv_kernel", int(best[1])); ctx.set_option("gemv_rows", int(best.split("r")[1]))
    ctx.set_option("profile_gemv", 1)
    x, h, r = ctx.cg(b, tol=0.0, maxit=40)
    out["cg_fixed40"] = {"ips": r.iterations / r.seconds_loop, "gemv_frac": r.seconds_gemv / r.seconds_loop,
                         "hist0": h[:3].tolist()}
    print(out["cg_fixed40"], flush=True)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open(f"gpurun_out/explore_{n}.json", "w"), indent=1)
