"""Diagnosis of the shared-device layouts: one subprocess per case (bounded), prints
status, iterations, error vs the oracle and wall time per case as JSON lines."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import json, sys, time
sys.path.insert(0, %r)
sys.path.insert(0, %r + "/tests")
import numpy as np
import paper_1511_07174_b200 as ks, synth, oracle
case, P = sys.argv[1], int(sys.argv[2])
_Ctx = ks.Context
class _C(_Ctx):
    def __init__(self, *a, **k):
        super().__init__(*a, **k)
        self.set_option("join_timeout_ms", 15000)
ks.Context = _C
out = {"case": case, "P": P}
t0 = time.time()
try:
    if case.startswith("bs"):
        n = int(case[2:])
        A, b = synth.gdd(n, 4)
        xo, ho, ro = oracle.bicgstab(A, b, tol=1e-10)
        with ks.Context(n, devices=[0] * P) as c:
            c.load_rows(A)
            for tiny in (0, 1):
                c.set_option("tiny", tiny)
                x, h, r = c.bicgstab(b, tol=1e-10)
                out[f"tiny{tiny}"] = [r.status, r.iterations, ro.iterations,
                                      float(np.linalg.norm(x - xo) / np.linalg.norm(xo))]
    elif case.startswith("x0"):
        n = int(case[2:])
        A = synth.random_spd(n, 10.0, 1)
        b = np.random.default_rng(0).standard_normal(n)
        x0 = np.random.default_rng(1).standard_normal(n)
        xo, ho, ro = oracle.cg(A, b, x0=x0, tol=1e-10)
        with ks.Context(n, devices=[0] * P) as c:
            c.load_rows(A)
            for tiny in (0, 1):
                c.set_option("tiny", tiny)
                x, h, r = c.cg(b, x0=x0, tol=1e-10)
                out[f"tiny{tiny}"] = [r.status, r.iterations, ro.iterations,
                                      float(np.linalg.norm(x - xo) / np.linalg.norm(xo))]
            y = c.matvec(x0)
            out["matvec_err"] = float(np.max(np.abs(y - A @ x0)))
    elif case.startswith("gm"):
        n = int(case[2:])
        A, b = synth.gdd(n, 16)
        xo, ho, ro = oracle.gmres(A, b, tol=1e-10, restart=30)
        with ks.Context(n, devices=[0] * P) as c:
            c.load_rows(A)
            for pers in (0, 1):
                c.set_option("persistent", pers)
                x, h, r = c.gmres(b, tol=1e-10, restart=30)
                out[f"pers{pers}"] = [r.status, r.iterations, ro.iterations,
                                      float(np.linalg.norm(x - xo) / np.linalg.norm(xo))]
    elif case.startswith("cg"):
        n = int(case[2:])
        A, c_, b = synth.gspd(n, 1e4)
        xo, ho, ro = oracle.cg(A, b, tol=1e-10)
        with ks.Context(n, devices=[0] * P) as c:
            c.generate("spd", seed=synth.SEED, table=c_)
            c.set_option("persistent", 1)
            x, h, r = c.cg(b, tol=1e-10)
            out["cg"] = [r.status, r.iterations, ro.iterations,
                         float(np.linalg.norm(x - xo) / np.linalg.norm(xo))]
except Exception as e:
    out["error"] = repr(e)[:400]
out["s"] = round(time.time() - t0, 2)
print(json.dumps(out))
''' % (ROOT, ROOT)

cases = sys.argv[1:] or ["bs1024:2", "bs1024:4", "x064:2", "x01000:2", "gm1024:2", "cg2048:4", "cg4096:4"]
for cs in cases:
    case, P = cs.split(":")
    try:
        r = subprocess.run([sys.executable, "-c", CHILD, case, P], capture_output=True, text=True, timeout=150)
        line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else json.dumps(
            {"case": case, "P": int(P), "rc": r.returncode, "stderr": r.stderr[-600:]})
    except subprocess.TimeoutExpired:
        line = json.dumps({"case": case, "P": int(P), "timeout": 150})
    print(line, flush=True)
