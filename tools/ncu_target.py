"""Small driver for one ncu capture: runs a solve whose kernel of interest is
then selected with ncu -k.  Usage: python tools/ncu_target.py {k1t|small|gmres}"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1511_07174_b200 as ks  # noqa: E402
import synth  # noqa: E402

what = sys.argv[1]
if what == "k1t":                          # BiCG at n = 65536: K1T launches
    with ks.Context(65536) as ctx:
        b = ctx.generate("dd", seed=synth.SEED, kd=16)
        ctx.set_option("true_residual", 0)
        ctx.bicg(b, tol=0.0, maxit=3, hist=False)
elif what == "small":                      # C1 CG on the small-n kernel
    n = 1024
    with ks.Context(n) as ctx:
        b = ctx.generate("spd", seed=synth.SEED, table=synth.spd_table(n, 1e3))
        ctx.set_option("true_residual", 0)
        ctx.cg(b, tol=0.0, maxit=64, hist=False)
elif what == "gmres":                      # GMRES(30) cycle kernel at n = 65536
    with ks.Context(65536) as ctx:
        b = ctx.generate("dd", seed=synth.SEED, kd=16)
        ctx.set_option("true_residual", 0)
        ctx.gmres(b, tol=0.0, restart=30, maxit=30, hist=False)
print("ok", what)
