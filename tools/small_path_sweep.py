"""NEXT-2 small-n path: us/iteration of the small shared-memory kernels (small=1)
vs the general persistent kernels (small=0), CG and BiCGSTAB, FP64 and FP32, 1 GPU.
Also the solve time to tol (1e-10 FP64, 1e-5 FP32).  -> gpurun_out/small_path.json"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1511_07174_b200 as ks
import synth

res = []
ns = [int(v) for v in sys.argv[1].split(",")] if len(sys.argv) > 1 else [512, 1024, 2048, 4096, 8192]
for dtype, tol in (("f64", 1e-10), ("f32", 1e-5)):
    for n in ns:
        for method, kind in (("cg", "spd"), ("bicgstab", "dd")):
            with ks.Context(n, dtype=dtype) as ctx:
                b = ctx.generate(kind, seed=synth.SEED, table=synth.spd_table(n, 1e3) if kind == "spd" else None,
                                 kd=16)
                ctx.set_option("true_residual", 0)
                for small in (0, 1):
                    ctx.set_option("small", small)
                    getattr(ctx, method)(b, tol=0.0, maxit=64, hist=False)
                    K = 1000 if method == "cg" else 500
                    _, _, r = getattr(ctx, method)(b, tol=0.0, maxit=K, hist=False)
                    _, _, r2 = getattr(ctx, method)(b, tol=tol)
                    row = {"dtype": dtype, "n": n, "method": method, "small": small,
                           "iters_timed": r.iterations, "us_per_iter": 1e6 * r.seconds_loop / max(1, r.iterations),
                           "solve_ms": 1e3 * r2.seconds_total, "solve_loop_ms": 1e3 * r2.seconds_loop,
                           "iters_to_tol": r2.iterations, "status": r2.status}
                    print(json.dumps(row), flush=True)
                    res.append(row)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/small_path.json", "w"), indent=1)
