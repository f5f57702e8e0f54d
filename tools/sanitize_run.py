"""Small solves in every kernel mode, for compute-sanitizer (one GPU, n <= 1100)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1511_07174_b200 as ks
import synth
for n in (1024, 777):
    A = synth.gspd(n, 1e3)[0] if n % 2 == 0 else synth.random_spd(n, 100.0, 1)
    D = synth.gdd(n, 4)[0]
    b = synth.rhs(n)
    for opts in ({"persistent": 1}, {"persistent": 0}, {"persistent": 0, "use_graphs": 1},
                 {"persistent": 0, "gemv_rows": 8}, {"persistent": 0, "gemv_split": 3}):
        with ks.Context(n) as c1, ks.Context(n) as c2:
            c1.load_rows(A); c2.load_rows(D)
            for k, v in opts.items():
                c1.set_option(k, v); c2.set_option(k, v)
            x, h, r = c1.cg(b, tol=1e-10, maxit=60)
            x2, h2, r2 = c2.bicgstab(b, x0=np.ones(n), tol=1e-10, maxit=20)
            y = c1.matvec(b)
            print(n, opts, r.iterations, r2.iterations, flush=True)
print("sanitize run OK")
