"""C1 latency vs the tiny kernels' CTA count (KS_TINY_GRID, tuning): one process per
setting (the grid is memoised per context), CG 200 and BiCGSTAB 30 fixed iterations
on the C1 matrices, best of 5 per setting.  One JSON line per setting."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import json, sys
sys.path.insert(0, %r)
import paper_1511_07174_b200 as ks, synth
n = 1024
out = {}
with ks.Context(n) as c:
    b = c.generate("spd", seed=synth.SEED, table=synth.spd_table(n, 1e3))
    c.cg(b, tol=0.0, maxit=2, hist=False)
    out["cg_us"] = min(1e6 * c.cg(b, tol=0.0, maxit=200, hist=False)[2].seconds_loop / 200 for _ in range(5))
with ks.Context(n) as c:
    b = c.generate("dd", seed=synth.SEED, kd=16)
    c.bicgstab(b, tol=0.0, maxit=2, hist=False)
    out["bs_us"] = min(1e6 * c.bicgstab(b, tol=0.0, maxit=30, hist=False)[2].seconds_loop / 30 for _ in range(5))
print(json.dumps(out))
''' % ROOT

for g in sys.argv[1:] or ["148", "128", "112", "96", "74"]:
    env = dict(os.environ, KS_TINY_GRID=g)
    r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True, timeout=300)
    rec = {"grid": int(g), "rc": r.returncode}
    if r.returncode == 0:
        rec.update(json.loads(r.stdout.strip().splitlines()[-1]))
    else:
        rec["err"] = r.stderr[-400:]
    print(json.dumps(rec), flush=True)
