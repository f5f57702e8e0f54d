"""torchrun worker: one process per GPU, torch's NCCL communicator borrowed by
ks_create_rank.  Runs CG and BiCGSTAB and writes per-rank results as JSON."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist
import paper_1511_07174_b200 as ks
import synth

n = int(sys.argv[1]); outdir = sys.argv[2]
local = int(os.environ["LOCAL_RANK"]); torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
rank, world = dist.get_rank(), dist.get_world_size()
res = {"rank": rank, "world": world}
with ks.Context.from_process_group(n) as ctx:
    assert ctx.nranks == world
    b = ctx.generate("spd", seed=synth.SEED, table=synth.spd_table(n, 1e4))
    x, h, r = ctx.cg(b, tol=1e-10)
    res["cg"] = {"x": x.tolist(), "h": h.tolist(), "it": r.iterations, "status": r.status, "true": r.true_relres}
    y = ctx.matvec(b)
    res["matvec"] = y.tolist()
with ks.Context.from_process_group(n) as ctx:
    b = ctx.generate("dd", seed=synth.SEED, kd=16)
    x, h, r = ctx.bicgstab(b, tol=1e-10)
    res["bs"] = {"x": x.tolist(), "h": h.tolist(), "it": r.iterations, "status": r.status,
                 "half": r.half_step_exit, "true": r.true_relres}
    # load_rows path: every rank passes only its own rows
    A, bb = synth.gdd(n, 4) if n <= 4096 else (None, None)
    if A is not None:
        with ks.Context.from_process_group(n) as c2:
            r0, r1 = c2.row_range(rank)
            c2.load_rows(A[r0:r1], r0)
            x2, h2, rr = c2.bicgstab(bb, tol=1e-10)
            res["bs_loaded"] = {"x": x2.tolist(), "h": h2.tolist(), "it": rr.iterations}
# fused NVLink collectives (default) vs NCCL allgathers: bitwise identical
with ks.Context.from_process_group(n) as ctx:
    b = ctx.generate("dd", seed=synth.SEED, kd=16)
    res["fused_effective"] = ctx.get_option("fused_comm")
    res["persistent_effective"] = ctx.get_option("persistent")
    x, h, r = ctx.bicgstab(b, tol=1e-10)          # default: persistent + fused
    res["bs_persistent"] = {"x": x.tolist(), "h": h.tolist(), "it": r.iterations}
    ctx.set_option("persistent", 0)                # multi-kernel: fused vs NCCL bitwise
    for mode in (1, 0):
        ctx.set_option("fused_comm", mode)
        x, h, r = ctx.bicgstab(b, tol=1e-10)
        res[f"bs_mode{mode}"] = {"x": x.tolist(), "h": h.tolist(), "it": r.iterations}
    # GMRES(20): persistent cycle kernel with fused exchanges (default) in this mode
    ctx.set_option("persistent", 2)
    ctx.set_option("fused_comm", 1)
    x, h, r = ctx.gmres(b, tol=1e-10, restart=20)
    res["gmres"] = {"x": x.tolist(), "h": h.tolist(), "it": r.iterations}
json.dump(res, open(os.path.join(outdir, f"dist_{n}_r{rank}.json"), "w"))
dist.destroy_process_group()
