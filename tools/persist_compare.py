"""Persistent cooperative kernels vs one-kernel-per-step (P = 1): us/iteration."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1511_07174_b200 as ks
import synth
rows = []
for n in [int(v) for v in (sys.argv[1:] or ["1024", "4096", "16384", "65536"])]:
    for method, kind in (("cg", "spd"), ("bicgstab", "dd")):
        with ks.Context(n) as ctx:
            b = ctx.generate(kind, seed=synth.SEED, table=synth.spd_table(n, 1e3) if kind == "spd" else None, kd=16)
            ctx.set_option("true_residual", 0)
            K = 400 if n <= 4096 else (100 if n <= 16384 else 20)
            for mode, graphs in ((0, 0), (0, 1), (1, 0)):
                ctx.set_option("persistent", mode); ctx.set_option("use_graphs", graphs)
                getattr(ctx, method)(b, tol=0.0, maxit=K // 4, hist=False)
                _, _, r = getattr(ctx, method)(b, tol=0.0, maxit=K, hist=False)
                _, _, r2 = getattr(ctx, method)(b, tol=1e-10)
                row = {"n": n, "method": method, "persistent": mode, "graphs": graphs,
                       "us_per_iter": 1e6 * r.seconds_loop / K, "solve_ms_to_tol": 1e3 * r2.seconds_total,
                       "iters_to_tol": r2.iterations, "launches": r.kernel_launches}
                print(json.dumps(row), flush=True); rows.append(row)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(rows, open("gpurun_out/persist_compare.json", "w"), indent=1)
