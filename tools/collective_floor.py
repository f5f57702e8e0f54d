"""Collective latency floor under torchrun: NCCL allgather
of 64 KiB - 4 MiB totals and 8-32 B scalar allreduce / allgather, CUDA events,
median of 50 after 10 warm-ups.  The per-iteration communication floor."""
import json, os, sys
import torch, torch.distributed as dist
local = int(os.environ["LOCAL_RANK"]); torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
rank, world = dist.get_rank(), dist.get_world_size()
rows = []
def bench(fn, reps=50):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    t = torch.tensor([ts[len(ts) // 2]], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.item()
for total in (64 << 10, 256 << 10, 512 << 10, 1 << 20, 4 << 20):
    per = total // 8 // world
    src = torch.zeros(per, dtype=torch.float64, device="cuda")
    dst = torch.zeros(per * world, dtype=torch.float64, device="cuda")
    us = bench(lambda: dist.all_gather_into_tensor(dst, src))
    rows.append({"op": "allgather", "total_bytes": total, "P": world, "us": us})
for nbytes in (8, 32):
    v = torch.zeros(nbytes // 8, dtype=torch.float64, device="cuda")
    rows.append({"op": "allreduce", "bytes": nbytes, "P": world, "us": bench(lambda: dist.all_reduce(v))})
    g = torch.zeros(nbytes // 8 * world, dtype=torch.float64, device="cuda")
    rows.append({"op": "allgather_scalars", "bytes_per_rank": nbytes, "P": world,
                 "us": bench(lambda: dist.all_gather_into_tensor(g, v))})
if rank == 0:
    for r in rows:
        print(json.dumps(r), flush=True)
    os.makedirs("gpurun_out", exist_ok=True)
    json.dump(rows, open(f"gpurun_out/collective_floor_p{world}.json", "w"), indent=1)
dist.destroy_process_group()
