"""torchrun worker for the solve-start rendezvous tests: the last rank
reaches each solve `delay` seconds after its peers.

    dist_skew.py n delay join_timeout_ms outdir

Writes per-rank {status, iterations} of one CG and one BiCGSTAB solve."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist
import paper_1511_07174_b200 as ks
import synth

n, delay, tmo, outdir = int(sys.argv[1]), float(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
local = int(os.environ["LOCAL_RANK"]); torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
rank, world = dist.get_rank(), dist.get_world_size()
res = {"rank": rank}
ctx = ks.Context.from_process_group(n)
b = ctx.generate("spd", seed=synth.SEED, table=synth.spd_table(n, 1e3))
ctx.set_option("join_timeout_ms", tmo)
for name in ("cg", "bicgstab"):
    if rank == world - 1:
        time.sleep(delay)
    try:
        x, h, r = getattr(ctx, name)(b, tol=1e-10)
        res[name] = {"status": r.status, "it": r.iterations, "x0": float(x[0])}
    except ks.KsError as e:
        res[name] = {"status": e.status, "error": str(e)}
        break                       # the context is poisoned after a peer timeout
json.dump(res, open(os.path.join(outdir, f"skew_r{rank}.json"), "w"))
# every rank outlives its peers' kernels: a rank whose solve failed early must keep
# its exchange buffers mapped until the late rank's kernel has given up too
torch.cuda.synchronize()
dist.barrier()
ctx.close()
dist.destroy_process_group()
