"""A/B of the persistent GEMV phase's row reductions: per tile (KS_GEMV_DEFER=0) vs
deferred to the end of the phase (1).  One subprocess per setting; us per iteration
(best of 3) for CG and BiCGSTAB at n = 65536 (default shape), 16384 and 8192 (default
and one-row tiles).  One JSON line per (setting, case)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import json, sys
sys.path.insert(0, %r)
import paper_1511_07174_b200 as ks, synth
out = []
for n, rows, its in ((65536, 0, 20), (16384, 0, 200), (16384, 1, 200), (8192, 0, 400), (8192, 1, 400)):
    for method in ("cg", "bicgstab"):
        with ks.Context(n) as c:
            b = c.generate("spd", seed=synth.SEED, table=synth.spd_table(n, 1e4)) if method == "cg" else \
                c.generate("dd", seed=synth.SEED, kd=16)
            c.set_option("true_residual", 0)
            c.set_option("small", 0)
            c.set_option("gemv_rows", rows)
            fn = c.cg if method == "cg" else c.bicgstab
            k = its if method == "cg" else its // 2
            fn(b, tol=0.0, maxit=3, hist=False)
            us = min(1e6 * fn(b, tol=0.0, maxit=k, hist=False)[2].seconds_loop / k for _ in range(3))
            gbs = (8.0 * n * n * (1 if method == "cg" else 2)) / (us * 1e-6) / 1e9
            out.append({"n": n, "rows": rows, "method": method, "us_per_iter": round(us, 2), "GBps": round(gbs, 1)})
print(json.dumps(out))
''' % ROOT
for rep in (1, 2):
    for d in ("0", "1"):
        env = dict(os.environ, KS_GEMV_DEFER=d)
        r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True, timeout=900)
        if r.returncode != 0:
            print(json.dumps({"defer": d, "rep": rep, "err": r.stderr[-500:]}), flush=True)
            continue
        for rec in json.loads(r.stdout.strip().splitlines()[-1]):
            rec.update({"defer": int(d), "rep": rep})
            print(json.dumps(rec), flush=True)
