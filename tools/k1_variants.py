"""K1 shapes at n = 65536 (and 32768), 1 GPU: the LDG stream at R=2/U=4 (default),
R=4/U=2 and R=4/U=4 (round 1 also timed a TMA ring, since removed:
profiles/r01_k1_variants.json).  ks_time_matvec, best of 3 x 10.
-> gpurun_out/k1_variants.json"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1511_07174_b200 as ks
import synth
res = []
for n in (65536, 32768):
    with ks.Context(n) as ctx:
        ctx.generate("dd", seed=synth.SEED, kd=16, want_b=False)
        for variant, R, U in ((1, 0, 0), (1, 4, 2), (1, 4, 4)):
            ctx.set_option("gemv_kernel", variant)
            ctx.set_option("gemv_rows", R)
            ctx.set_option("gemv_unroll", U)
            t = min(ctx.time_matvec(10) for _ in range(3))
            row = {"n": n, "variant": "LDG" if variant == 1 else "TMA", "R": R or 2, "U": (U or 4) if variant == 1 else None,
                   "ms": t * 1e3, "GBps": 8.0 * n * n / t / 1e9}
            print(json.dumps(row), flush=True)
            res.append(row)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/k1_variants.json", "w"), indent=1)
