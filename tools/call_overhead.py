"""Per-call overhead of ks_cg / ks_bicgstab (bench `e2e` = one call per method per
step): where do the microseconds between the device-loop iteration time and a
maxit = 1 call on host buffers go?  One process, P = 1 (or torchrun for P > 1).

Reports, per method: device loop time per iteration (maxit = K in one call), the
per-call time with device buffers and with pinned host buffers (maxit = 1), and a
CUPTI timeline (torch.profiler sees every kernel / memcpy of libks.so) of a few
host-buffer calls: kernel and copy durations and the idle gaps between them.

    python tools/call_overhead.py [--size 65536] [--calls 20] [--out gpurun_out/call_overhead.json]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_1511_07174_b200 as ks  # noqa: E402
import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=65536)
    ap.add_argument("--calls", type=int, default=20)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "call_overhead.json"))
    a = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", 1))
    rank = int(os.environ.get("RANK", 0))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    n, K = a.size, a.calls
    stream = torch.cuda.current_stream()

    def mk():
        if world > 1:
            return ks.Context.from_process_group(n)
        return ks.Context.from_rank(n, 0, 1, None, local, stream.cuda_stream)

    def sync():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    out = {"n": n, "P": world}
    ctxs = {"cg": mk(), "bicgstab": mk()}
    bcg = ctxs["cg"].generate("spd", seed=synth.SEED, table=synth.spd_table(n, 1e4))
    bbs = ctxs["bicgstab"].generate("dd", seed=synth.SEED, kd=16)
    for c in ctxs.values():
        c.set_option("true_residual", 0)
    for meth, b in (("cg", bcg), ("bicgstab", bbs)):
        c = ctxs[meth]
        fn = getattr(c, meth)
        bd = torch.from_numpy(b).to(dev)
        xd = torch.empty(n, dtype=torch.float64, device=dev)
        bh = torch.from_numpy(b).pin_memory()
        xh = torch.empty(n, dtype=torch.float64).pin_memory()
        hh = torch.empty(max(K, 1), dtype=torch.float64).pin_memory()
        fn(bd, tol=0.0, maxit=3, out=xd, hist=False)
        sync()
        r = {}
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        _, _, rep = fn(bd, tol=0.0, maxit=K, out=xd, hist=False)
        e1.record(stream)
        sync()
        r["loop_ms_per_iter"] = rep.seconds_loop * 1e3 / K
        r["one_call_K_iters_ms_per_iter"] = e0.elapsed_time(e1) / K
        for tag, bb, xx, hs in (("dev", bd, xd, False), ("host", bh, xh, hh[:1])):
            sync()
            t0 = time.perf_counter()
            e0.record(stream)
            inside = 0.0
            for _ in range(K):
                inside += fn(bb, tol=0.0, maxit=1, out=xx, hist=hs)[2].seconds_total
            e1.record(stream)
            sync()
            r[f"call_{tag}_ms_wall"] = (time.perf_counter() - t0) * 1e3 / K
            r[f"call_{tag}_ms_inside_c"] = inside * 1e3 / K     # ks_cg's own wall time (C side)
            r[f"call_{tag}_ms_events"] = e0.elapsed_time(e1) / K
        # maxit = 0: the call's fixed cost without any iteration
        sync()
        t0 = time.perf_counter()
        inside = 0.0
        for _ in range(K):
            inside += fn(bh, tol=0.0, maxit=0, out=xh, hist=hh[:1])[2].seconds_total
        sync()
        r["call_host_maxit0_ms_wall"] = (time.perf_counter() - t0) * 1e3 / K
        r["call_host_maxit0_ms_inside_c"] = inside * 1e3 / K
        # CUPTI timeline of 3 host-buffer calls
        from torch.profiler import ProfilerActivity, profile
        sync()
        with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
            for _ in range(3):
                fn(bh, tol=0.0, maxit=1, out=xh, hist=hh[:1])
            torch.cuda.synchronize()
        ev = []
        for e in prof.events():
            if e.device_type == torch.autograd.DeviceType.CUDA:
                ev.append((e.time_range.start, e.time_range.end, e.name))
        ev.sort()
        items = []
        for i, (s, t, nm) in enumerate(ev):
            gap = (s - ev[i - 1][1]) if i else 0.0
            items.append({"name": nm[:60], "us": round(t - s, 2), "gap_before_us": round(gap, 2)})
        r["timeline_3_calls"] = items
        trace = os.path.join(os.path.dirname(a.out), f"call_overhead_{meth}_P{world}_r{rank}.json")
        os.makedirs(os.path.dirname(trace), exist_ok=True)
        prof.export_chrome_trace(trace)
        out[meth] = r
    if rank == 0:
        os.makedirs(os.path.dirname(a.out), exist_ok=True)
        with open(a.out, "w") as f:
            json.dump(out, f, indent=1)
        print(json.dumps({m: {k: v for k, v in out[m].items() if k != "timeline_3_calls"}
                          for m in ("cg", "bicgstab")}))
    for c in ctxs.values():
        c.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
