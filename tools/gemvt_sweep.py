"""K1T (A^T x) shape sweep at n = 65536, 1 GPU; BiCG it/s for the default."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1511_07174_b200 as ks
import synth
n = 65536
res = []
with ks.Context(n) as ctx:
    b = ctx.generate("dd", seed=synth.SEED, kd=16)
    ctx.set_option("true_residual", 0); ctx.set_option("profile_gemv", 1)
    for shape in (104, 108, 116, 204, 208, 216, 404, 408):
        ctx.set_option("gemvt_shape", shape)
        ctx.bicg(b, tol=0.0, maxit=2, hist=False)
        _, _, r = ctx.bicg(b, tol=0.0, maxit=12, hist=False)
        t_k1t = 0
        row = {"shape": shape, "bicg_iters_per_s": 12 / r.seconds_loop,
               "avg_GBps_two_gemvs": 8.0 * n * n * r.gemv_launches / r.seconds_gemv / 1e9}
        print(json.dumps(row), flush=True); res.append(row)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/gemvt_sweep.json", "w"), indent=1)
