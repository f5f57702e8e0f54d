"""Multi-rank host logic on CPU (world sizes 2 and 8, gloo, 127.0.0.1).

The CUDA path's N > 1 schedule is: row-block partition
(`ks.partition` == ks_row_range), gather buffers in chunk layout whose tail slots
carry each rank's partial scalars, rank-ordered sums of those partials, and the
full-length direction vectors formed redundantly on every rank.  This test runs
that exact data flow with numpy on 2 gloo ranks (the GPU arithmetic is replaced by
numpy; the collectives by torch.distributed over gloo) and checks
  * every rank takes identical decisions and ends with identical x / history,
  * the result meets the north-star bars against the oracle,
  * row-sharded generation reassembles the full matrix bitwise.
"""
import os
import queue
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import paper_1511_07174_b200 as ks
import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class Layout:
    """Mirror of ks::Layout (csrc/ks_internal.h): chunk = round_up(mmax,32)+32."""

    def __init__(self, n, P, rank):
        self.n, self.P, self.rank = n, P, rank
        self.parts = ks.partition(n, P)
        mmax = max(e - b for b, e in self.parts)
        self.pslot = (mmax + 31) // 32 * 32
        self.chunk = self.pslot + 32
        self.r0, self.r1 = self.parts[rank]

    def gather(self, local, partials):
        """In-place allgather of [slice || partials] (ncclAllGather in the library)."""
        buf = np.zeros(self.chunk)
        buf[: local.size] = local
        buf[self.pslot: self.pslot + len(partials)] = partials
        out = torch.zeros(self.P * self.chunk, dtype=torch.float64)
        dist.all_gather_into_tensor(out, torch.from_numpy(buf))
        G = out.numpy().reshape(self.P, self.chunk)
        full = np.concatenate([G[g, : e - b] for g, (b, e) in enumerate(self.parts)])
        sums = [sum(G[g, self.pslot + k] for g in range(self.P)) for k in range(len(partials))]
        return full, sums   # rank-ordered sums, identical on every rank

    def scalars(self, partials):
        out = torch.zeros(self.P * 4, dtype=torch.float64)
        buf = np.zeros(4)
        buf[: len(partials)] = partials
        dist.all_gather_into_tensor(out, torch.from_numpy(buf))
        S = out.numpy().reshape(self.P, 4)
        return [sum(S[g, k] for g in range(self.P)) for k in range(len(partials))]


def cg_model(L, A_loc, b, tol, maxit):
    """CG schedule of ks_solvers.cpp::run_cg with numpy arithmetic."""
    r_loc = b[L.r0:L.r1].copy()
    x_loc = np.zeros(L.r1 - L.r0)
    nb = np.sqrt(b @ b)
    r_full, (rho,) = L.gather(r_loc, [r_loc @ r_loc])
    p = r_full.copy()
    hist, k_done = [], 0
    if np.sqrt(rho) / nb <= tol:
        return x_loc, hist, 0
    for k in range(1, maxit + 1):
        q = A_loc @ p
        (sigma,) = L.scalars([p[L.r0:L.r1] @ q])
        alpha = rho / sigma
        x_loc += alpha * p[L.r0:L.r1]
        r_loc -= alpha * q
        r_full, (rho1,) = L.gather(r_loc, [r_loc @ r_loc])
        rel = np.sqrt(rho1) / nb
        hist.append(rel)
        k_done = k
        if rel <= tol:
            break
        p = r_full + (rho1 / rho) * p
        rho = rho1
    return x_loc, hist, k_done


def bicgstab_model(L, A_loc, b, tol, maxit):
    """BiCGSTAB schedule of ks_solvers.cpp::run_bicgstab (replicated-vector form)."""
    r_loc = b[L.r0:L.r1].copy()
    rhat = r_loc.copy()
    x_loc = np.zeros(L.r1 - L.r0)
    nb = np.sqrt(b @ b)
    r_full, (rho, rr) = L.gather(r_loc, [rhat @ r_loc, r_loc @ r_loc])
    hist = []
    if np.sqrt(rr) / nb <= tol:
        return x_loc, hist, 0, False
    rho_old = alpha = omega = 1.0
    p = np.zeros(L.n)
    v_full = np.zeros(L.n)
    for i in range(1, maxit + 1):
        if i >= 2:
            rel = np.sqrt(rr) / nb
            hist.append(rel)
            if rel <= tol:
                return x_loc, hist, i - 1, False
        beta = (rho / rho_old) * (alpha / omega)
        p = r_full.copy() if i == 1 else r_full + beta * (p - omega * v_full)
        v_loc = A_loc @ p
        v_full, (g,) = L.gather(v_loc, [rhat @ v_loc])
        alpha = rho / g
        s = r_full - alpha * v_full
        srel = np.sqrt(s @ s) / nb                      # full length, redundant
        if srel <= tol:
            hist.append(srel)
            x_loc += alpha * p[L.r0:L.r1]
            return x_loc, hist, i, True
        t_loc = A_loc @ s
        s_loc = s[L.r0:L.r1]
        ts, tt = L.scalars([t_loc @ s_loc, t_loc @ t_loc])
        omega = ts / tt
        x_loc += alpha * p[L.r0:L.r1] + omega * s_loc
        r_loc = s_loc - omega * t_loc
        rho_old = rho
        r_full, (rho, rr) = L.gather(r_loc, [rhat @ r_loc, r_loc @ r_loc])
    hist.append(np.sqrt(rr) / nb)
    return x_loc, hist, maxit, False


def _worker(rank, world, port, n, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        L = Layout(n, world, rank)
        A, c, b = synth.gspd(n, 1e3)
        A_loc = synth.gspd_rows(n, c, synth.SEED, L.r0, L.r1)       # row-sharded generation
        assert np.array_equal(A_loc, A[L.r0:L.r1])
        x_loc, hist, k = cg_model(L, A_loc, b, 1e-10, 10 * n)
        x_full, _ = L.gather(x_loc, [])
        D, bd = synth.gdd(n, 16)
        D_loc = synth.gdd_rows(n, 16, synth.SEED, L.r0, L.r1)
        assert np.array_equal(D_loc, D[L.r0:L.r1])
        y_loc, bh, bk, half = bicgstab_model(L, D_loc, bd, 1e-10, 10 * n)
        y_full, _ = L.gather(y_loc, [])
        q.put((rank, x_full, np.array(hist), k, y_full, np.array(bh), bk, half))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 256), (2, 1000), (8, 1002)])
def test_multi_rank_schedule_gloo(world, n):
    """world = 8 is the driver's largest scaling run; n = 1002 gives ragged shards."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = []
    while len(res) < world:                     # fail fast if a worker dies
        try:
            res.append(q.get(timeout=5))
        except queue.Empty:
            dead = [p.exitcode for p in procs if p.exitcode not in (None, 0)]
            assert not dead, f"worker exited with {dead}"
    res.sort(key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    r0 = res[0]
    for rr in res[1:]:                          # identical decisions and results on every rank
        for a, b in zip(r0[1:], rr[1:]):
            if isinstance(a, np.ndarray):
                assert np.array_equal(a, b)
            else:
                assert a == b
    A, c, b = synth.gspd(n, 1e3)
    xo, ho, ro = oracle.cg(A, b, tol=1e-10)
    _, x, h, k = r0[0], r0[1], r0[2], r0[3]
    assert abs(k - ro.iterations) <= 2
    m = min(50, len(h), len(ho))
    assert np.all(np.abs(h[:m] - ho[:m]) <= 1e-8 * ho[:m] + 1e-14)
    assert np.linalg.norm(x - xo) <= 1e-9 * np.linalg.norm(xo)
    D, bd = synth.gdd(n, 16)
    yo, hyo, ryo = oracle.bicgstab(D, bd, tol=1e-10)
    y, bh, bk, half = r0[4], r0[5], r0[6], r0[7]
    assert abs(bk - ryo.iterations) <= 2 and half == ryo.half_step_exit
    m = min(50, len(bh), len(hyo))
    assert np.all(np.abs(bh[:m] - hyo[:m]) <= 1e-8 * hyo[:m] + 1e-12)
    assert np.linalg.norm(y - yo) <= 1e-9 * np.linalg.norm(yo)


def test_layout_mirrors_header_partition():
    for n, P in [(10, 3), (65536, 8), (2050, 4)]:
        L = Layout(n, P, P - 1)
        assert L.chunk % 32 == 0 and L.pslot >= max(e - b for b, e in L.parts)
        assert L.parts == ks.partition(n, P)
