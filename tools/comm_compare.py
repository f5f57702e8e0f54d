"""Fused NVLink collectives vs NCCL allgathers at P ranks (torchrun): it/s and
K1 time per method at n (default 65536)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.distributed as dist
import paper_1511_07174_b200 as ks
import synth
n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
local = int(os.environ["LOCAL_RANK"]); torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
rank, world = dist.get_rank(), dist.get_world_size()
rows = []
for method, kind in (("cg", "spd"), ("bicgstab", "dd")):
    with ks.Context.from_process_group(n) as ctx:
        b = ctx.generate(kind, seed=synth.SEED, table=synth.spd_table(n, 1e4) if kind == "spd" else None, kd=16)
        ctx.set_option("true_residual", 0)
        for mode in (0, 1, 0, 1):
            for prof in (1, 0):
                ctx.set_option("fused_comm", mode); ctx.set_option("profile_gemv", prof)
                K = 40 if method == "cg" else 20
                getattr(ctx, method)(b, tol=0.0, maxit=4, hist=False)
                _, _, r = getattr(ctx, method)(b, tol=0.0, maxit=K, hist=False)
                t = torch.tensor([r.seconds_loop, r.seconds_gemv], dtype=torch.float64, device="cuda")
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                row = {"method": method, "P": world, "n": n, "fused": ctx.get_option("fused_comm"), "profile": prof,
                       "iters_per_s": K / t[0].item(),
                       "gemv_ms": 1e3 * t[1].item() / max(1, r.gemv_launches) if prof else None,
                       "overhead_us_per_iter": 1e6 * (t[0].item() - t[1].item()) / K if prof else None}
                if rank == 0:
                    print(json.dumps(row), flush=True); rows.append(row)
if rank == 0:
    json.dump(rows, open(f"gpurun_out/comm_compare_p{world}.json", "w"), indent=1)
dist.destroy_process_group()
