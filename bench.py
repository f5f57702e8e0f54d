"""Benchmark of the dense FP64 CG / BiCGSTAB hot path (BASELINE.json metric
"CG/BiCGSTAB iters/s & GEMV HBM GB/s vs peak, n=65536 FP64, 1/2/4/8 B200").

Workload (config C3/C3' of SURVEY.md sec.8(d).3): n = 65536, FP64, A row-block
sharded over N GPUs (strong scaling).  Two matrices are resident in HBM:
G-SPD(65536, kappa=1e4) for CG and G-DD(65536, kd=16) for BiCGSTAB (seed
151107174, generated on the device).  One STEP = one CG iteration + one BiCGSTAB
iteration = every row of sec.8(a) (3 GEMVs, 3 x 8 n^2 / N bytes per GPU).
value = steps/s for the whole job.  Timed: K steps = ks_cg(maxit=K) +
ks_bicgstab(maxit=K) with tol = 0 (fixed length), inputs resident on the device,
bracketed by barrier + synchronize, CUDA events on the stream the library runs
on (torch's current stream, borrowed), max over ranks.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--size 65536]
    torchrun --nproc-per-node N bench.py --gpus N ...

--impl reference times the CPU oracle (oracle/, the only baseline this paper
has) on the same full workload -- K oracle iterations of each method after W
warm-up iterations, all host cores, plus one single-thread step -- on rank 0 only.
The matrices are stored on the host when RAM allows (2 x 34.4 GB at n = 65536),
else generated row by row on the fly.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "CG/BiCGSTAB iters/s & GEMV HBM GB/s vs peak, n=65536 FP64, 1/2/4/8 B200"
UNIT = "steps/s (step = 1 CG iter + 1 BiCGSTAB iter)"
SEED = 151107174
NOMINAL_HBM = 8000.0   # GB/s, north star's "~8 TB/s"


def workload(n: int) -> str:
    """The measured problem, identical in both arms (ours and --impl reference)."""
    return (f"C3/C3': n={n} FP64 dense, CG on G-SPD(kappa=1e4) + BiCGSTAB on G-DD(kd=16), "
            f"seed 151107174, tol=0 fixed length, 1 step = 1 CG + 1 BiCGSTAB iteration")


def env_int(k, d):
    return int(os.environ.get(k, d))


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ----------------------------------------------------------------- clocks

def environment(local: int) -> dict:
    """GPU / driver / NCCL / torch versions and memory clock."""
    import torch
    env = {"gpu": torch.cuda.get_device_name(local), "torch": torch.__version__,
           "cuda_runtime": torch.version.cuda}
    try:
        v = torch.cuda.nccl.version()
        env["nccl"] = ".".join(str(x) for x in v) if isinstance(v, tuple) else str(v)
    except Exception:
        pass
    try:
        out = subprocess.run(["nvidia-smi", f"--id={local}", "--query-gpu=driver_version,clocks.max.mem,clocks.mem",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=10).stdout
        drv, mmax, mem = [x.strip() for x in out.strip().split(",")]
        env.update(driver=drv, mem_max_mhz=float(mmax), mem_mhz=float(mem))
    except Exception:
        pass
    return env


def topology(world: int, local: int) -> dict:
    """Rank -> GPU map and the peer topology the fused exchange runs over (the
    fused path makes no NCCL call per iteration, so NCCL's own communicator lines
    say little about it)."""
    import torch
    import torch.distributed as dist
    me = {"rank": int(os.environ.get("RANK", 0)), "local_rank": local,
          "device": torch.cuda.get_device_name(local),
          "pci": torch.cuda.get_device_properties(local).pci_bus_id
          if hasattr(torch.cuda.get_device_properties(local), "pci_bus_id") else None}
    ranks = [me]
    if world > 1:
        ranks = [None] * world
        dist.all_gather_object(ranks, me)
    nd = torch.cuda.device_count()
    p2p = {f"{i}->{j}": bool(torch.cuda.can_device_access_peer(i, j))
           for i in range(nd) for j in range(nd) if i != j}
    links = None
    try:
        out = subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True,
                             timeout=10).stdout
        rows = [ln.split() for ln in out.splitlines() if ln.startswith("GPU")]
        links = {r[0]: r[1:1 + nd] for r in rows[:nd]} if rows else None
    except Exception:
        pass
    return {"world_size": world, "ranks": ranks, "visible_gpus": nd,
            "peer_access_all_pairs": all(p2p.values()) if p2p else None,
            "nvidia_smi_topo": links}


class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        time.sleep(0.25)
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out = ""
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def clocks_bad(c):
    bad = {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
    if bad & set(c.get("reasons", [])):
        return True
    if c.get("sm_mhz") and c.get("sm_max_mhz") and not c["reasons"]:
        return c["sm_mhz"] < 0.5 * c["sm_max_mhz"]
    return False


# ------------------------------------------------------------ CPU oracle

def host_info() -> dict:
    info = {"nproc": os.cpu_count()}
    try:
        with open("/proc/cpuinfo") as f:
            names = [ln.split(":", 1)[1].strip() for ln in f if ln.startswith("model name")]
        info["cpu_model"] = names[0] if names else None
    except OSError:
        pass
    try:
        with open("/proc/meminfo") as f:
            for ln in f:
                k, v = ln.split(":", 1)
                if k in ("MemTotal", "MemAvailable"):
                    info[k] = int(v.split()[0]) * 1024
    except OSError:
        pass
    return info


def oracle_full_steps(n: int, steps: int, warmup: int, threads: int, one_thread: bool = True) -> dict:
    """Times the CPU oracle AS IT STANDS on the full bench workload: the oracle's
    own CG (or_cg) and BiCGSTAB (or_bicgstab) run `steps` iterations each (tol = 0,
    fixed length) on G-SPD(n, 1e4) and G-DD(n, 16) -- a step is one CG + one
    BiCGSTAB iteration, 3 full n x n GEMVs and all the vector work.  The matrices
    are stored on the host (expanded by the oracle's generator on all cores) when
    RAM allows, else the oracle generates every row on the fly.  `threads` = the
    row-parallel OpenMP variant (each row sum stays sequential: bitwise the
    1-thread oracle); with one_thread, one further step runs on a single thread
    (PAPER.md:95's "serial version [that] uses one CPU")."""
    import oracle
    import synth
    info = host_info()
    need = 2 * 8.0 * n * n
    stored = info.get("MemAvailable", 0) > 1.25 * need + 16e9
    t_gen = time.perf_counter()
    specs = {"cg": synth.spec("spd", n, kappa=1e4, seed=SEED), "bicgstab": synth.spec("dd", n, kd=16, seed=SEED)}
    mats = {k: oracle.gen_rows(s, 0, n, threads=threads) if stored else None for k, s in specs.items()}
    t_gen = time.perf_counter() - t_gen

    def op(k, th):
        return oracle.Operator(mats[k], threads=th) if stored else oracle.Operator(gen=specs[k], threads=th)

    b = {"cg": synth.rhs(n, SEED), "bicgstab": synth.rhs(n, SEED)}
    ops = {k: op(k, threads) for k in specs}
    if warmup > 0:
        oracle.cg(ops["cg"], b["cg"], tol=0.0, maxit=warmup)
        oracle.bicgstab(ops["bicgstab"], b["bicgstab"], tol=0.0, maxit=warmup)
    t0 = time.perf_counter()
    _, _, r1 = oracle.cg(ops["cg"], b["cg"], tol=0.0, maxit=steps)
    t1 = time.perf_counter()
    _, _, r2 = oracle.bicgstab(ops["bicgstab"], b["bicgstab"], tol=0.0, maxit=steps)
    t2 = time.perf_counter()
    assert r1.iterations == steps and r2.iterations == steps, (r1, r2)
    sec = (t2 - t0) / steps
    out = {"value": 1.0 / sec, "unit": UNIT, "cores": threads, "kind": "oracle",
           "sample": f"the full workload, not a sample: the oracle's own CG and BiCGSTAB, {steps} "
                     f"iterations each (tol=0) on G-SPD(n={n},1e4) and G-DD(n={n},16), "
                     f"{'host-stored rows' if stored else 'rows generated on the fly'}, "
                     f"row-parallel on {threads} threads (sequential FP64 row sums); "
                     f"{warmup} warm-up iterations per method untimed",
           "seconds_per_step": sec, "timed_steps": steps,
           "cg_iters_per_s": steps / (t1 - t0), "bicgstab_iters_per_s": steps / (t2 - t1),
           "matrix": "stored" if stored else "on-the-fly", "generate_s": t_gen, "host": info}
    if one_thread:
        o1 = {k: op(k, 1) for k in specs}
        s0 = time.perf_counter()
        oracle.cg(o1["cg"], b["cg"], tol=0.0, maxit=1)
        s1 = time.perf_counter()
        oracle.bicgstab(o1["bicgstab"], b["bicgstab"], tol=0.0, maxit=1)
        s2 = time.perf_counter()
        out["one_thread"] = {"value": 1.0 / (s2 - s0), "unit": UNIT, "cores": 1,
                             "seconds_per_step": s2 - s0, "cg_seconds_per_iter": s1 - s0,
                             "bicgstab_seconds_per_iter": s2 - s1, "timed_steps": 1,
                             "gemv_GBps": 3 * 8.0 * n * n / (s2 - s0) / 1e9}
    return out


def run_reference(args):
    rank = env_int("RANK", 0)
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    n = args.n
    t0 = time.perf_counter()
    cpu = oracle_full_steps(n, args.steps, args.warmup, threads, one_thread=True)
    wall = time.perf_counter() - t0
    cpu["fits_in_run"] = cpu["seconds_per_step"] * args.steps <= wall
    line = {"impl": "reference", "metric": METRIC, "value": cpu["value"], "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 / cpu["value"], "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload(n), "n": n,
                       "parallelism": "CPU oracle on the host cores, rank 0 only"},
            "cpu_baseline": cpu,
            "e2e": {"value": cpu["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "wall_s": wall}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------- our path

def run_ours(args):
    # stdout carries exactly one JSON line: C-level prints (NCCL banner, ...) go to stderr
    json_out = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    import torch
    import torch.distributed as dist

    import paper_1511_07174_b200 as ks
    import synth

    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local = env_int("LOCAL_RANK", 0)
    if args.gpus != world:
        raise SystemExit(f"bench: --gpus {args.gpus} but WORLD_SIZE={world} ranks were launched")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    n, K, W = args.n, args.steps, args.warmup
    stream = torch.cuda.current_stream()

    def mk():
        if world > 1:
            return ks.Context.from_process_group(n)
        return ks.Context.from_rank(n, 0, 1, None, local, stream.cuda_stream)

    def barrier():
        if world > 1:
            dist.barrier()

    def allmax(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def allsum(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t)
        return float(t.item())

    # C1 latency extra (n = 1024, tiny kernels), measured first: a latency-bound kernel
    # timed right after seconds of full-HBM streaming would see the power-capped clock
    c1_latency = None
    if world == 1 and not args.no_extras:
        with ks.Context.from_rank(1024, 0, 1, None, local, stream.cuda_stream) as c1:
            bt = c1.generate("spd", seed=SEED, table=synth.spd_table(1024, 1e3))
            c1.cg(bt, tol=0.0, maxit=2, hist=False)
            _, _, r1 = c1.cg(bt, tol=0.0, maxit=200, hist=False)
            _, _, r1t = c1.cg(bt, tol=1e-10, hist=False)
        with ks.Context.from_rank(1024, 0, 1, None, local, stream.cuda_stream) as c1:
            bd1 = c1.generate("dd", seed=SEED, kd=16)
            c1.bicgstab(bd1, tol=0.0, maxit=2, hist=False)
            _, _, r2 = c1.bicgstab(bd1, tol=0.0, maxit=30, hist=False)
        c1_latency = {
            "cg_us_per_iter": 1e6 * r1.seconds_loop / r1.iterations,
            "bicgstab_us_per_iter": 1e6 * r2.seconds_loop / r2.iterations,
            "cg_iters_to_tol_1e-10": r1t.iterations,
            "kernel": "k_cg_tiny / k_bs_tiny (A in registers, LL exchange)"}

    t_gen = time.perf_counter()
    cg_ctx, bs_ctx = mk(), mk()
    table = synth.spd_table(n, 1e4, SEED)
    b_cg = cg_ctx.generate("spd", seed=SEED, table=table)
    b_bs = bs_ctx.generate("dd", seed=SEED, kd=16)
    t_gen = time.perf_counter() - t_gen
    for c in (cg_ctx, bs_ctx):
        c.set_option("true_residual", 0)
        c.set_option("profile_gemv", 1)
        c.set_option("fused_comm", 1 if args.comm == "fused" else 0)
    comm_mode = "fused NVLink peer stores" if cg_ctx.get_option("fused_comm") else \
        ("none (P=1)" if world == 1 else "NCCL allgather")
    if args.kernels == "multi":
        for c in (cg_ctx, bs_ctx):
            c.set_option("persistent", 0)
    persistent = bool(cg_ctx.get_option("persistent"))
    small = persistent and world == 1 and 8 * n <= 32768      # KS_OPT_SMALL auto bound
    dominant = ("k_cg_small + k_bs_small (small-n persistent kernels, vectors in shared memory)" if small
                else "k_cg_persist + k_bs_persist (persistent cooperative whole-iteration kernels: "
                "3 GEMVs + fused vector phases per step)" if persistent else "k1_gemv_ldg (K1 GEMV)")
    row_b, row_e = cg_ctx.row_range(rank)
    m = row_e - row_b

    bd_cg = torch.from_numpy(b_cg).to(dev)
    bd_bs = torch.from_numpy(b_bs).to(dev)
    xd = torch.empty(n, dtype=torch.float64, device=dev)

    def device_steps(k):
        _, _, r1 = cg_ctx.cg(bd_cg, tol=0.0, maxit=k, out=xd, hist=False)
        _, _, r2 = bs_ctx.bicgstab(bd_bs, tol=0.0, maxit=k, out=xd, hist=False)
        assert r1.iterations == k and r2.iterations == k, (r1, r2)
        return r1, r2

    device_steps(W)                               # warm-up (W >= 3 steps)
    torch.cuda.synchronize()

    def timed():
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(local) as cs:
            e0.record(stream)
            r1, r2 = device_steps(K)
            e1.record(stream)
            torch.cuda.synchronize()
        barrier()
        return e0.elapsed_time(e1) * 1e-3, r1, r2, cs.summary()

    sec, r_cg, r_bs, clocks = timed()
    remeasured = False
    if clocks_bad(clocks):
        sec, r_cg, r_bs, clocks = timed()
        remeasured = True
    sec = allmax(sec)
    cg_loop, bs_loop = allmax(r_cg.seconds_loop), allmax(r_bs.seconds_loop)
    gemv_s = allmax(r_cg.seconds_gemv + r_bs.seconds_gemv)
    gemv_n = r_cg.gemv_launches + r_bs.gemv_launches
    launches = allsum(float(r_cg.kernel_launches + r_bs.kernel_launches))

    # e2e: the public API with HOST (pinned) buffers.  Every step is one user call per
    # method (ks_cg / ks_bicgstab, maxit = 1, x0 = 0): H2D of b and D2H of x and the
    # step's residual-history entry inside the timed region, every step.
    bh_cg = torch.from_numpy(b_cg).pin_memory()
    bh_bs = torch.from_numpy(b_bs).pin_memory()
    xh = torch.empty(n, dtype=torch.float64).pin_memory()
    hh = torch.empty(max(K, 1), dtype=torch.float64).pin_memory()

    def e2e_region(per_step: bool) -> float:
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        if per_step:
            for _ in range(K):
                cg_ctx.cg(bh_cg, tol=0.0, maxit=1, out=xh, hist=hh[:1])
                bs_ctx.bicgstab(bh_bs, tol=0.0, maxit=1, out=xh, hist=hh[:1])
        else:
            cg_ctx.cg(bh_cg, tol=0.0, maxit=K, out=xh, hist=hh)
            bs_ctx.bicgstab(bh_bs, tol=0.0, maxit=K, out=xh, hist=hh)
        e1.record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        barrier()
        return allmax(max(e0.elapsed_time(e1) * 1e-3, wall))

    e2e_s = e2e_region(True)
    e2e_solve_s = e2e_region(False)

    # extras (outside the timed region, one GPU only): multi-RHS CG and BiCGSTAB on the
    # resident matrices (8 right-hand sides share each pass over A)
    # and the C1 latency path (n = 1024, tiny register-resident kernels)
    extras = None
    if world == 1 and not args.no_extras:
        extras = {}
        B = np.column_stack([b_cg] + [synth.rhs(n, SEED + j) for j in range(1, 8)])
        cg_ctx.cg_multi(B, tol=0.0, maxit=2, hist=False)
        _, _, rm = cg_ctx.cg_multi(B, tol=0.0, maxit=K, hist=False)
        ips_m = K / rm[0].seconds_loop
        extras["multi_rhs_cg"] = {
            "nrhs": 8, "iters_per_s": ips_m, "rhs_iters_per_s": 8 * ips_m,
            "A_stream_GBps": 8.0 * n * n * ips_m / 1e9, "vs_single_rhs_cg": 8 * ips_m / (K / cg_loop),
            "kernel": "k_cgm<8,8,128> (TMA 2-D tensor-map loads, producer warp + 7 consumer warps, FP64 skinny GEMM)"}
        Bb = np.column_stack([b_bs] + [synth.rhs(n, SEED + j) for j in range(1, 8)])
        bs_ctx.bicgstab_multi(Bb, tol=0.0, maxit=2, hist=False)
        _, _, rb8 = bs_ctx.bicgstab_multi(Bb, tol=0.0, maxit=min(K, 10), hist=False)
        ips_b = min(K, 10) / rb8[0].seconds_loop
        extras["multi_rhs_bicgstab"] = {
            "nrhs": 8, "iters_per_s": ips_b, "rhs_iters_per_s": 8 * ips_b,
            "A_stream_GBps": 2 * 8.0 * n * n * ips_b / 1e9, "vs_single_rhs_bicgstab": 8 * ips_b / (K / bs_loop),
            "kernel": "k_bsm<8,8,128> (both GEMMs of an iteration TMA-fed and shared by 8 columns)"}
        extras["c1_latency"] = c1_latency

    # roofline of the dominant kernel (K1 GEMV): algorithmic bytes 8*m*n per launch
    gemv_avg = gemv_s / max(1, gemv_n)
    achieved = 8.0 * m * n / gemv_avg / 1e9
    peak, peak_kind = measured_peak()
    traffic = None
    tp = os.path.join(ROOT, "profiles", "gemv_traffic.json")
    if os.path.exists(tp):
        try:
            t = json.load(open(tp))
            if int(t.get("n", -1)) == n and int(t.get("P", -1)) == world and \
                    t.get("persistent", False) == persistent:
                traffic = t.get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    topo = topology(world, local)          # collective: every rank takes part
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            cpu = oracle_full_steps(n, args.cpu_steps, 1, os.cpu_count() or 1, one_thread=True)
        value = K / sec
        T_roof = lambda g: g * 8.0 * n * n / world / (NOMINAL_HBM * 1e9) + \
            g * 8.0 * n * (world - 1) / world / 0.9e12
        cg_ips, bs_ips = K / cg_loop, K / bs_loop
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
            "warmup": W, "ms_per_step": 1e3 * sec / K, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (G-SPD kappa=1e4 + G-DD kd=16, seed 151107174, generated on device)",
            "config": {"workload": workload(n), "n": n,
                       "parallelism": f"row-block over {world} GPU(s) (P={world})",
                       "collectives": comm_mode,
                       "kernels": "persistent cooperative" if persistent else "one kernel per step",
                       "l2": f"no flush needed: resident inputs {2 * 8 * m * n / 1e9:.1f} GB/GPU "
                             f">> 126 MB L2"},
            "per_method": {
                "cg_iters_per_s": cg_ips, "bicgstab_iters_per_s": bs_ips,
                "cg_frac_of_roofline_8TBps": cg_ips * T_roof(1),
                "bicgstab_frac_of_roofline_8TBps": bs_ips * T_roof(2),
                "cg_target_80pct_1gpu": 186.3, "bicgstab_target_80pct_1gpu": 93.1},
            "roofline": {"bound": "hbm", "kernel": dominant, "achieved": achieved,
                         "peak": peak, "peak_kind": f"{peak_kind} copy GB/s (MEASURED_PEAKS.json)",
                         "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                         "algorithmic_bytes_per_gemv": 8.0 * m * n,
                         "avg_ms_per_gemv": gemv_avg * 1e3, "frac_of_nominal_8TBps": achieved / NOMINAL_HBM,
                         "gemv_share_of_step": gemv_s / sec},
            "e2e": {"value": K / e2e_s, "unit": UNIT,
                    "h2d_bytes_per_step": 2 * 8 * n, "d2h_bytes_per_step": 2 * 8 * (n + 1),
                    "bytes_scope": "per rank (b in, x and the history entry out, both methods)",
                    "how": "K steps, each = ks_cg + ks_bicgstab with maxit=1, x0=0, host pinned b/x/hist"},
            "e2e_solve": {"value": K / e2e_solve_s, "unit": UNIT,
                          "how": "one ks_cg + one ks_bicgstab call of K iterations each, host pinned "
                                 "b/x/hist (copies amortised over K)"},
            "gpu_launches": int(launches),
            "clocks": clocks, "remeasured": remeasured,
            "cpu_baseline": cpu,
            "extras": extras,
            "generate_s": t_gen,
            "env": environment(local),
            "topology": topo,
        }
        json_out.write(json.dumps(line) + "\n")
        json_out.flush()
    cg_ctx.close()
    bs_ctx.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=env_int("WORLD_SIZE", 1))
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--size", dest="n", type=int, default=65536)   # not "--n": torchrun would take it as an abbreviation of its own options
    ap.add_argument("--cpu-steps", type=int, default=3)      # cpu_baseline leg: full oracle steps
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--comm", choices=["fused", "nccl"], default="fused")
    ap.add_argument("--kernels", choices=["persistent", "multi"], default="persistent")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        return relaunch(args.gpus)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


def relaunch(n: int) -> int:
    """`python bench.py --gpus N` without a launcher: re-execute this same command
    under torch.distributed.run with one process per GPU (the driver's own launch
    line), so N ranks always run -- never a silent one-GPU run."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.abspath(__file__), *sys.argv[1:]]
    print(f"bench: launching {n} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    return subprocess.call(cmd)


if __name__ == "__main__":
    sys.exit(main())
