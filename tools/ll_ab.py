"""A/B of the persistent kernels' handovers over P GPUs (one process): KS_OPT_LL_XCHG
0 (stores + fence + epoch flag) vs 1 (LL words), us per iteration (best of 3) for CG
and BiCGSTAB at n = 16384 and 65536, and the strong-scaling efficiency against the same
kernels on one GPU.  One JSON line per (n, P, method, ll)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1511_07174_b200 as ks  # noqa: E402
import synth  # noqa: E402

ngpu = torch.cuda.device_count()
for n, its in ((16384, 300), (65536, 40)):
    base = {}
    for P in [1] + [q for q in (2, 4, 8) if q <= ngpu]:
        for method in ("cg", "bicgstab"):
            with ks.Context(n, ngpus=P) as c:
                if method == "cg":
                    b = c.generate("spd", seed=synth.SEED, table=synth.spd_table(n, 1e4))
                else:
                    b = c.generate("dd", seed=synth.SEED, kd=16)
                c.set_option("true_residual", 0)
                for ll in ((0, 1) if P > 1 else (1,)):
                    c.set_option("ll_xchg", ll)
                    fn = c.cg if method == "cg" else c.bicgstab
                    k = its if method == "cg" else its // 2
                    fn(b, tol=0.0, maxit=3, hist=False)
                    us = min(1e6 * fn(b, tol=0.0, maxit=k, hist=False)[2].seconds_loop / k for _ in range(3))
                    if P == 1:
                        base[method] = us
                    rec = {"n": n, "P": P, "method": method, "ll": ll, "us_per_iter": round(us, 2),
                           "efficiency": round(base[method] / (P * us), 4)}
                    print(json.dumps(rec), flush=True)
