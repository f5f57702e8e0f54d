"""K1 tile-shape sweep (rows R x unroll U, LDG stream) at n = 65536, 1 GPU."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1511_07174_b200 as ks
import synth
n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
res = []
with ks.Context(n) as ctx:
    ctx.generate("dd", seed=synth.SEED, kd=16, want_b=False)
    for R in (2, 4, 8):
        for U in (1, 2, 4, 8):
            if R * U > 32:
                continue
            ctx.set_option("gemv_rows", R); ctx.set_option("gemv_unroll", U)
            t = min(ctx.time_matvec(10) for _ in range(3))
            row = {"R": R, "U": U, "ms": t * 1e3, "GBps": 8.0 * n * n / t / 1e9}
            print(json.dumps(row), flush=True); res.append(row)
    ctx.set_option("gemv_rows", 0); ctx.set_option("gemv_unroll", 0)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/gemv_sweep.json", "w"), indent=1)
