"""Multi-RHS CG throughput (ks_cg_multi) at n = 65536 FP64 on one GPU: for
nrhs = 1, 2, 4, 8, a fixed-length solve (tol = 0) of `iters` iterations; reports
iterations/s, right-hand-side-iterations/s and the A-stream GB/s of the TMA-fed
skinny GEMM (8 n^2 bytes per iteration, algorithmic), next to single-RHS ks_cg.

    python tools/multi_rhs_bench.py [--size 65536] [--iters 20]
    torchrun --nproc-per-node P tools/multi_rhs_bench.py      (row blocks over P GPUs)
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=65536)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--method", choices=["cg", "bicgstab"], default="cg")
    a = ap.parse_args()
    import paper_1511_07174_b200 as ks
    import synth
    n, K = a.size, a.iters
    world = int(os.environ.get("WORLD_SIZE", 1))
    rank = int(os.environ.get("RANK", 0))
    if world > 1:
        import torch
        import torch.distributed as dist
        local = int(os.environ["LOCAL_RANK"])
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    out = print if rank == 0 else (lambda *x, **y: None)
    bs = a.method == "bicgstab"
    single = "bicgstab" if bs else "cg"
    multi = "bicgstab_multi" if bs else "cg_multi"
    g = 2 if bs else 1                               # GEMMs per iteration
    with (ks.Context.from_process_group(n) if world > 1 else ks.Context(n)) as ctx:
        b = ctx.generate("dd", seed=synth.SEED, kd=16) if bs else \
            ctx.generate("spd", seed=synth.SEED, table=synth.spd_table(n, 1e4))
        ctx.set_option("true_residual", 0)
        getattr(ctx, single)(b, tol=0.0, maxit=2, hist=False)
        _, _, r1 = getattr(ctx, single)(b, tol=0.0, maxit=K, hist=False)
        single_ips = K / r1.seconds_loop
        out(json.dumps({"P": world, "nrhs": 1, "kernel": "ks_" + single, "iters_per_s": single_ips,
                        "GBps_per_gpu": g * 8.0 * n * n * single_ips / world / 1e9}), flush=True)
        for nrhs in (1, 2, 4, 8):
            B = np.column_stack([b] + [synth.rhs(n, synth.SEED + j) for j in range(1, nrhs)])
            getattr(ctx, multi)(B, tol=0.0, maxit=2, hist=False)
            X, h, r = getattr(ctx, multi)(B, tol=0.0, maxit=K, hist=False)
            t = r[0].seconds_loop
            ips = K / t
            out(json.dumps({"P": world, "nrhs": nrhs, "kernel": "ks_" + multi, "iters_per_s": ips,
                              "rhs_iters_per_s": nrhs * ips, "GBps_per_gpu": g * 8.0 * n * n * ips / world / 1e9,
                              "speedup_vs_single_rhs": nrhs * ips / single_ips,
                              "statuses": [q.status for q in r]}), flush=True)


if __name__ == "__main__":
    main()
    if int(os.environ.get("WORLD_SIZE", 1)) > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
