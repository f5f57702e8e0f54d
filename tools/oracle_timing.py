"""Oracle timing on the GPU box's host: the plain oracle on
1 thread (the paper's 'serial version that uses one CPU') and its
row-parallel GEMV on all cores (bitwise equal).  Full C1 / C1b solves; per-GEMV
time at n = 32768 / 65536 from row samples (extrapolated, labelled)."""
import json, os, platform, subprocess, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
import synth

out = {"nproc": os.cpu_count(), "platform": platform.platform()}
try:
    out["cpu_model"] = [l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name")][0]
    out["mem_total_kB"] = int([l.split()[1] for l in open("/proc/meminfo") if l.startswith("MemTotal")][0])
except Exception:
    pass
A, c, b = synth.gspd(1024, 1e3)
t = time.perf_counter(); x, h, r = oracle.cg(A, b, tol=1e-10); dt = time.perf_counter() - t
out["C1_cg_1thread"] = {"seconds": dt, "iterations": r.iterations, "us_per_iter": 1e6 * dt / r.iterations}
for kd in (4, 16):
    D, bd = synth.gdd(1024, kd)
    t = time.perf_counter(); x, h, r = oracle.bicgstab(D, bd, tol=1e-10); dt = time.perf_counter() - t
    out[f"C1b_bicgstab_kd{kd}_1thread"] = {"seconds": dt, "iterations": r.iterations}
for n in (32768, 65536):
    rows = 512
    Ar = oracle.gen_rows(synth.spec("dd", n, kd=16), n // 2, rows)
    xv = synth.rhs(n)
    y = np.empty(rows)
    L = oracle.lib()
    res = {}
    for th in (1, os.cpu_count()):
        best = 1e9
        for _ in range(3):
            t = time.perf_counter()
            L.or_gemv(rows, n, oracle._p(Ar), n, oracle._p(xv), oracle._p(y), th)
            best = min(best, time.perf_counter() - t)
        per_gemv = best * n / rows
        res[f"threads_{th}"] = {"gemv_seconds_extrapolated": per_gemv, "GBps": 8.0 * n * n / per_gemv / 1e9,
                                "cg_iters_per_s": 1.0 / per_gemv, "bicgstab_iters_per_s": 0.5 / per_gemv}
    out[f"n{n}"] = {"sample": f"{rows} rows of G-DD(n={n},16), best of 3, x n/rows", **res}
print(json.dumps(out, indent=1))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/oracle_timing.json", "w"), indent=1)
