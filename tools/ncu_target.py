"""Small driver for one ncu capture: runs a solve whose kernel of interest is
then selected with ncu -k.
Usage: python tools/ncu_target.py {k1t|small|gmres|tiny|tinybs|multi8|persist|persistbs}"""
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
elif what in ("tiny", "tinybs"):           # C1 on the register-resident tiny kernels
    n = 1024
    with ks.Context(n) as ctx:
        if what == "tiny":
            b = ctx.generate("spd", seed=synth.SEED, table=synth.spd_table(n, 1e3))
            ctx.set_option("true_residual", 0)
            ctx.cg(b, tol=0.0, maxit=200, hist=False)
        else:
            b = ctx.generate("dd", seed=synth.SEED, kd=16)
            ctx.set_option("true_residual", 0)
            ctx.bicgstab(b, tol=0.0, maxit=30, hist=False)
elif what == "multi8":                     # multi-RHS CG, 8 right-hand sides, n = 65536
    import numpy as np
    n = 65536
    with ks.Context(n) as ctx:
        b = ctx.generate("spd", seed=synth.SEED, table=synth.spd_table(n, 1e4))
        B = np.column_stack([b] + [synth.rhs(n, synth.SEED + j) for j in range(1, 8)])
        ctx.cg_multi(B, tol=0.0, maxit=4, hist=False)
elif what in ("persist", "persistbs"):     # the bench's persistent kernels, n = 65536
    n = 65536
    with ks.Context(n) as ctx:
        ctx.set_option("true_residual", 0)
        if what == "persist":
            b = ctx.generate("spd", seed=synth.SEED, table=synth.spd_table(n, 1e4))
            ctx.cg(b, tol=0.0, maxit=6, hist=False)
        else:
            b = ctx.generate("dd", seed=synth.SEED, kd=16)
            ctx.bicgstab(b, tol=0.0, maxit=3, hist=False)
print("ok", what)
