"""Out-of-bounds-write check (run with KS_GUARD=1): every solver path and kernel mode
on small ragged systems, 1 GPU and (if present) 2-4 GPUs; prints the number of
corrupted guard zones (must be 0)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1511_07174_b200 as ks
import synth

assert os.environ.get("KS_GUARD") == "1", "run with KS_GUARD=1"
ngpu = torch.cuda.device_count()
total = 0
modes = [{}, {"persistent": 0}, {"persistent": 0, "use_graphs": 1}, {"persistent": 0, "gemv_rows": 8},
         {"persistent": 0, "gemv_split": 3}, {"small": 0}, {"poll_batch": 3}, {"gemv_rows": 4, "gemv_unroll": 2},
         {"tiny": 0}]
for P in [p for p in (1, 2, 4) if p <= ngpu]:
    for n in (300, 777, 1024, 2050):            # n <= 1024: the tiny kernels by default
        A = synth.random_spd(n, 100.0, 1)
        D = synth.gdd(n, 4, seed=synth.SEED2)[0]
        b = synth.rhs(n)
        for opts in modes:
            for dtype in ("f64", "f32"):
                with ks.Context(n, ngpus=P, dtype=dtype) as c1, ks.Context(n, ngpus=P, dtype=dtype) as c2:
                    c1.load_rows(A)
                    c2.load_rows(D)
                    for k, v in opts.items():
                        c1.set_option(k, v)
                        c2.set_option(k, v)
                    tol = 1e-10 if dtype == "f64" else 1e-5
                    c1.cg(b, tol=tol, maxit=80)
                    c2.bicgstab(b, tol=tol, maxit=40)
                    c1.matvec(b)
                    if dtype == "f64":
                        c1.cg(b, x0=np.ones(n), tol=tol, maxit=30)
                        c2.bicg(b, tol=tol, maxit=40)
                        c2.gmres(b, tol=tol, restart=7, maxit=40)
                        c2.matvec_t(b)
                        if not opts:                    # multi-RHS kernels (TMA GEMM), 3 columns
                            B = np.column_stack([b, synth.rhs(n, synth.SEED + 1), np.zeros(n)])
                            c1.cg_multi(B, tol=tol, maxit=30)
                            c2.bicgstab_multi(B, X0=1e-3 * np.ones((n, 3)), tol=tol, maxit=20)
                    v1, v2 = c1.check_guards(), c2.check_guards()
                    total = max(total, v1, v2)
                    if v1 or v2:
                        print("VIOLATION", P, n, opts, dtype, v1, v2, flush=True)
    print("P", P, "done", flush=True)
print("violations", total)
