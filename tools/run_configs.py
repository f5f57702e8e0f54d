"""Runs the concrete configs of SURVEY.md sec.8(d).3 (C1..C5) on 1 GPU or under
torchrun, one matrix resident at a time: fixed-length it/s (tol = 0), a
to-tolerance solve (iterations, true residual) and checks that hold at any size
(closed form for G-SPD).  Prints one JSON line per config (rank 0).

    python tools/run_configs.py C1 C2 C3 C3p C4
    torchrun --nproc-per-node 4 tools/run_configs.py C3 C3p C4 C5cg C5bs
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

CONFIGS = {
    "C1": ("cg", 1024, dict(kappa=1e3), 200),
    "C2": ("cg", 32768, dict(kappa=1e4), 100),
    "C3": ("bicgstab", 65536, dict(kd=16), 30),
    "C3p": ("cg", 65536, dict(kappa=1e4), 60),
    "C4": ("cg", 131072, dict(kappa=1e4), 20),
    "C5cg": ("cg", 262144, dict(kappa=1e4), 8),
    "C5bs": ("bicgstab", 262144, dict(kd=16), 4),
    "C3bicg": ("bicg", 65536, dict(kd=16), 30),       # NEXT-3: BiCG (A p and A^T pt)
    "C1bicg": ("bicg", 1024, dict(kd=16), 200),
    "C1bs": ("bicgstab", 1024, dict(kd=16), 30),        # C1b: converges at 34 (no breakdown at tol 0)
    "C3gmres": ("gmres", 65536, dict(kd=16), 30),     # NEXT-3: GMRES(30)
    "C1gmres": ("gmres", 1024, dict(kd=16), 200),
    "C2bs": ("bicgstab", 32768, dict(kd=16), 50),       # per-rank size of n = 65536 at P = 8 (P = 2)
    "C16cg": ("cg", 16384, dict(kappa=1e4), 200),
    "C16bs": ("bicgstab", 16384, dict(kd=16), 100),
}
NOMINAL = 8000e9


def main():
    import torch
    import torch.distributed as dist

    import paper_1511_07174_b200 as ks
    import synth

    world = int(os.environ.get("WORLD_SIZE", 1))
    rank = int(os.environ.get("RANK", 0))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    out = []
    for name in sys.argv[1:]:
        dtype = "f64"
        if name.endswith(":f32"):
            name, dtype = name[:-4], "f32"
        method, n, gp, K = CONFIGS[name]
        if world > 1:
            ctx = ks.Context.from_process_group(n, dtype=dtype)
        else:
            ctx = ks.Context.from_rank(n, 0, 1, None, local, torch.cuda.current_stream().cuda_stream,
                                       dtype=dtype)
        t0 = time.perf_counter()
        table = None
        if method == "cg":
            table = synth.spd_table(n, gp["kappa"])
            b = ctx.generate("spd", seed=synth.SEED, table=table)
        else:
            b = ctx.generate("dd", seed=synth.SEED, kd=gp["kd"])
        tgen = time.perf_counter() - t0
        solve = getattr(ctx, method)
        ctx.set_option("true_residual", 0)
        ctx.set_option("profile_gemv", 1)
        if "KS_PERSISTENT" in os.environ:                # comparisons: force the kernel mode
            ctx.set_option("persistent", int(os.environ["KS_PERSISTENT"]))
        if "KS_TINY" in os.environ:                      # comparisons: tiny kernels on / off
            ctx.set_option("tiny", int(os.environ["KS_TINY"]))
        if "KS_FUSED" in os.environ:                     # comparisons: fused vs NCCL exchange
            ctx.set_option("fused_comm", int(os.environ["KS_FUSED"]))
        solve(b, tol=0.0, maxit=2, hist=False)                     # warm-up
        _, _, r = solve(b, tol=0.0, maxit=K, hist=False)
        ips = r.iterations / r.seconds_loop
        g = 1 if method in ("cg", "gmres") else 2   # GEMVs per iteration
        m = ctx.row_range(rank)[1] - ctx.row_range(rank)[0]
        esz = 4.0 if dtype == "f32" else 8.0
        gemv_bw = esz * m * n * r.gemv_launches / max(r.seconds_gemv, 1e-12)
        t_roof = g * esz * n * n / world / NOMINAL + g * esz * n * (world - 1) / world / 0.9e12
        ctx.set_option("profile_gemv", 0)
        ctx.set_option("true_residual", 1)
        x, h, rt = solve(b, tol=1e-5 if dtype == "f32" else 1e-10)
        rec = {"config": name, "dtype": dtype, "method": method, "n": n, "P": world, "gen_s": tgen,
               "fixed_iters": K, "iters_run": r.iterations, "iters_per_s": ips, "us_per_iter": 1e6 / ips, "frac_roofline_8TBps": ips * t_roof,
               "gemv_GBps_per_gpu": gemv_bw / 1e9, "iters_to_tol": rt.iterations,
               "converged": rt.converged, "half_step_exit": rt.half_step_exit,
               "true_relres": rt.true_relres, "solve_s": rt.seconds_total, "hist0": h[:3].tolist()}
        if method == "cg" and rank == 0 and dtype == "f64":
            import oracle
            xcf = oracle.spd_exact_solve_ld(table, synth.SEED, b)
            rec["x_vs_closed_form"] = float(np.linalg.norm(x - xcf) / np.linalg.norm(xcf))
        ctx.close()
        del ctx
        torch.cuda.synchronize()
        if rank == 0:
            print(json.dumps(rec), flush=True)
            out.append(rec)
    if rank == 0:
        os.makedirs("gpurun_out", exist_ok=True)
        json.dump(out, open(f"gpurun_out/configs_p{world}.json", "w"), indent=1)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
