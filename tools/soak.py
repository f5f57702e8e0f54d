"""Soak test of the fused multi-GPU protocols: many back-to-back solves of random
size / method / maxit / tolerance on P GPUs (one context per (n, method) kept alive
and reused, so epochs, parities and the barrier counter roll over many solves).
Every result is checked: converged solves by the true residual, fixed-length runs by
bitwise repeatability.  Prints one summary JSON line."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1511_07174_b200 as ks
import synth

WORLD = int(os.environ.get("WORLD_SIZE", 1))          # torchrun: one process per GPU
if WORLD > 1:
    import torch.distributed as dist
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    P = WORLD
else:
    P = min(int(sys.argv[1]) if len(sys.argv) > 1 else 4, torch.cuda.device_count())
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 200
rng = np.random.default_rng(2024)
ctxs, fails, stats = {}, [], {"solves": 0, "iters": 0}
t0 = time.time()
for it in range(rounds):
    n = int(rng.choice([300, 777, 1024, 1000, 2049, 4096, 5003]))
    method = str(rng.choice(["cg", "bicgstab", "bicg", "gmres", "cg_multi", "bicgstab_multi"]))
    if method in ("cg", "cg_multi") and n % 2:
        n += 1                                   # G-SPD needs an even n
    key = (n, method)
    if key not in ctxs:
        c = ks.Context.from_process_group(n) if WORLD > 1 else ks.Context(n, ngpus=P)
        if method in ("cg", "cg_multi"):
            c.generate("spd", seed=synth.SEED, table=synth.spd_table(n, 1e3), want_b=False)
        else:
            c.generate("dd", seed=synth.SEED, kd=16, want_b=False)
        # 0 = auto: one launch per solve (tiny kernels at n <= 1024); else split launches
        c.set_option("poll_batch", int(rng.choice([0, 0, 1, 3, 16])))
        ctxs[key] = c
    c = ctxs[key]
    b = synth.rhs(n, synth.SEED + it)
    if method in ("cg_multi", "bicgstab_multi"):  # multi-RHS: a block of k right-hand sides
        k = int(rng.integers(1, 9))
        B = np.column_stack([synth.rhs(n, synth.SEED + 1000 * it + j) for j in range(k)])
        if rng.random() < 0.3:
            mx = int(rng.integers(1, 12))
            X1, _, r1 = getattr(c, method)(B, tol=0.0, maxit=mx)
            X2, _, r2 = getattr(c, method)(B, tol=0.0, maxit=mx)
            if not np.array_equal(X1, X2):
                fails.append({"round": it, "n": n, "method": method, "why": "not repeatable"})
        else:
            X, _, rs = getattr(c, method)(B, tol=1e-10)
            for j in range(k):
                res = np.linalg.norm(c.matvec(X[:, j]) - B[:, j]) / np.linalg.norm(B[:, j])
                if not (rs[j].converged and res <= 1e-8):
                    fails.append({"round": it, "n": n, "method": method, "why": f"col {j} true {res}"})
            stats["iters"] += max(q.iterations for q in rs)
        stats["solves"] += 1
        continue
    kw = {"restart": int(rng.choice([5, 20]))} if method == "gmres" else {}
    if method in ("cg", "bicgstab") and rng.random() < 0.25:
        kw["x0"] = rng.standard_normal(n)
    fixed = rng.random() < 0.3
    if fixed:
        mx = int(rng.integers(1, 12))
        x1, h1, r1 = getattr(c, method)(b, tol=0.0, maxit=mx, **kw)
        x2, h2, r2 = getattr(c, method)(b, tol=0.0, maxit=mx, **kw)
        if not (r1.iterations == r2.iterations and np.array_equal(x1, x2) and np.array_equal(h1, h2)):
            fails.append({"round": it, "n": n, "method": method, "why": "not repeatable"})
    else:
        x, h, r = getattr(c, method)(b, tol=1e-10, **kw)
        if not (r.converged and r.true_relres <= 1e-8):
            fails.append({"round": it, "n": n, "method": method, "why": f"status {r.status} true {r.true_relres}"})
        stats["iters"] += r.iterations
    stats["solves"] += 1
for c in ctxs.values():
    c.close()
if WORLD == 1 or dist.get_rank() == 0:
    print(json.dumps({"P": P, "mode": "torchrun" if WORLD > 1 else "single-process", "rounds": rounds,
                      "contexts": len(ctxs), "fails": fails, **stats, "seconds": time.time() - t0}))
if WORLD > 1:
    dist.destroy_process_group()
