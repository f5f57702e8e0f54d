"""Row-stride padding experiment (KS_LD_EXTRA), n = 65536, 1 GPU: K1 and persistent CG."""
import json, os, subprocess, sys
code = r'''
import json, os, sys
sys.path.insert(0, os.getcwd())
import paper_1511_07174_b200 as ks, synth
n = 65536
with ks.Context(n) as ctx:
    b = ctx.generate("spd", seed=synth.SEED, table=synth.spd_table(n, 1e4))
    k1 = min(ctx.time_matvec(10) for _ in range(3))
    ctx.set_option("true_residual", 0)
    ctx.cg(b, tol=0.0, maxit=4, hist=False)
    _, _, r = ctx.cg(b, tol=0.0, maxit=32, hist=False)
    print(json.dumps({"extra": int(os.environ.get("KS_LD_EXTRA", "0")), "ld": ctx.ld,
                      "k1_GBps": 8.0 * n * n / k1 / 1e9, "cg_iters_per_s": 32 / r.seconds_loop}))
'''
for extra in ("0", "1", "3", "0", "1", "3"):
    env = dict(os.environ, KS_LD_EXTRA=extra)
    print(subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True).stdout.strip(), flush=True)
