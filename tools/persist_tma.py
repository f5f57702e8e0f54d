"""Persistent kernels, LDG stream vs TMA ring GEMV phase (KS_OPT_GEMV_KERNEL 1 vs 2):
CG / BiCGSTAB it/s at n = 65536 (and 32768), FP64 and FP32, 1 GPU, alternating runs."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1511_07174_b200 as ks
import synth
res = []
for dtype in ("f64", "f32"):
    for n in (65536, 32768):
        for method, kind in (("cg", "spd"), ("bicgstab", "dd")):
            with ks.Context(n, dtype=dtype) as ctx:
                b = ctx.generate(kind, seed=synth.SEED, table=synth.spd_table(n, 1e4) if kind == "spd" else None, kd=16)
                ctx.set_option("true_residual", 0)
                K = 40 if method == "cg" else 20
                if n == 32768:
                    K *= 4
                for rep in range(3):
                    for variant in (1, 2):
                        ctx.set_option("gemv_kernel", variant)
                        getattr(ctx, method)(b, tol=0.0, maxit=4, hist=False)
                        _, _, r = getattr(ctx, method)(b, tol=0.0, maxit=K, hist=False)
                        gemvs = K * (2 if method == "bicgstab" else 1)
                        esz = 8 if dtype == "f64" else 4
                        row = {"dtype": dtype, "n": n, "method": method, "variant": "TMA" if variant == 2 else "LDG",
                               "rep": rep, "iters_per_s": K / r.seconds_loop,
                               "GBps": gemvs * esz * n * n / r.seconds_loop / 1e9}
                        print(json.dumps(row), flush=True)
                        res.append(row)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/persist_tma.json", "w"), indent=1)
