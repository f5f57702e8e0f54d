"""Multi-GPU parity (pin P13): P GPUs vs the oracle with the same bars, identical
results on every rank, and the two multi-GPU modes -- one process driving P GPUs
(ks_create, ncclCommInitAll + worker threads) and one process per GPU (torchrun,
torch's NCCL communicator borrowed through ks_create_rank)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu
ks = pytest.importorskip("paper_1511_07174_b200")
torch = pytest.importorskip("torch")

from test_gpu_parity import FLOOR_BS, bars, gemv_bound_check  # noqa: E402
from layouts import context, layouts, need  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def ngpu():
    return torch.cuda.device_count()


needs2 = pytest.mark.skipif("ngpu() < 2", reason="needs >= 2 GPUs (gpurun --gpus 2)")

# every multi-GPU test runs at each P the box has (the 8-GPU box of the driver's
# scaling step included); a P above the device count skips
PS = [2, 4, 8]


@pytest.mark.parametrize("lay", layouts())
def test_multi_gemv_and_cg(lay):
    P = need(lay)
    n = 2050   # uneven partition: first n mod P shards get one more row
    rng = np.random.default_rng(P)
    A = rng.standard_normal((n, n))
    x = rng.standard_normal(n)
    with context(n, lay) as ctx:
        assert ctx.nranks == P and ctx.local_gpus == P
        assert [ctx.row_range(g) for g in range(P)] == ks.partition(n, P)
        ctx.load_rows(A[:1000])
        ctx.load_rows(A[1000:], 1000)
        y = ctx.matvec(x)
    gemv_bound_check(A, x, y)
    n = 2048
    As, c, b = synth.gspd(n, 1e4)
    xo, ho, ro = oracle.cg(As, b, tol=1e-10)
    with context(n, lay) as ctx:
        ctx.generate("spd", seed=synth.SEED, table=c)
        xg, hg, rg = ctx.cg(b, tol=1e-10)
    bars(xg, hg, rg, xo, ho, ro)
    with ks.Context(n) as c1:
        c1.generate("spd", seed=synth.SEED, table=c)
        x1, h1, r1 = c1.cg(b, tol=1e-10)
    assert r1.iterations == rg.iterations


@pytest.mark.parametrize("lay", layouts(shared=()))
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_multi_small_cg_allgather_only(lay, dtype):
    """Small-n CG over P GPUs (k_cg_small_peer: one exchange of q slices and one grid
    barrier per iteration, all O(n) work redundant in shared memory) vs the oracle
    and vs the general fused kernels (small = 0): ragged n, x0, maxit, multi-launch."""
    P = need(lay)
    from test_gpu_parity import bars_f32
    for n in (1002, 4096):
        A, c, b = synth.gspd(n, 1e3)
        if dtype == "f32":
            xo, ho, ro = oracle.cg_f32(A, b, tol=1e-5)
        else:
            xo, ho, ro = oracle.cg(A, b, tol=1e-10)
        outs = []
        for small in (1, 0):
            with context(n, lay, dtype=dtype) as ctx:
                ctx.set_option("small", small)
                ctx.set_option("tiny", 0)     # the small-n kernels themselves (tiny: test_gpu_tiny.py)
                ctx.generate("spd", seed=synth.SEED, table=c, want_b=False)
                if dtype == "f32":
                    bb = b.astype(np.float32).astype(np.float64)
                    x, h, r = ctx.cg(bb, tol=1e-5)
                    bars_f32(x, h, r, xo, ho, ro)
                else:
                    x, h, r = ctx.cg(b, tol=1e-10)
                    bars(x, h, r, xo, ho, ro)
                    ctx.set_option("poll_batch", 7)
                    x2, h2, r2 = ctx.cg(b, tol=1e-10)
                    assert r2.iterations == r.iterations and np.array_equal(x2, x) and np.array_equal(h2, h)
                    x0 = np.random.default_rng(n).standard_normal(n)
                    xo0, ho0, ro0 = oracle.cg(A, b, x0=x0, tol=1e-30, maxit=9)
                    x9, h9, r9 = ctx.cg(b, x0=x0, tol=1e-30, maxit=9)
                    assert r9.status == ks.KS_EMAXIT and r9.iterations == 9
                    bars(x9, h9, r9, xo0, ho0, ro0, iters_tol=0)
                outs.append(r.iterations)
        assert abs(outs[0] - outs[1]) <= 2


@pytest.mark.parametrize("lay", layouts(shared=()))
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_multi_small_bicgstab_allgather_only(lay, dtype):
    """Small-n BiCGSTAB over P GPUs (k_bs_small_peer: v and t slices are the only
    exchanges, two grid barriers per iteration) vs the oracle and the general fused
    kernels: ragged n, half-step exit, maxit (in-kernel final test), x0, and a
    multi-launch solve (rhat and r handed over between launches)."""
    P = need(lay)
    from test_gpu_parity import bars_f32
    for n, kd in ((1003, 4), (4096, 16)):
        A, b = synth.gdd(n, kd)
        if dtype == "f32":
            xo, ho, ro = oracle.bicgstab_f32(A, b, tol=1e-5)
        else:
            xo, ho, ro = oracle.bicgstab(A, b, tol=1e-10)
        its = []
        for small in (1, 0):
            with context(n, lay, dtype=dtype) as ctx:
                ctx.set_option("small", small)
                ctx.set_option("tiny", 0)     # the small-n kernels themselves (tiny: test_gpu_tiny.py)
                ctx.load_rows(A)
                if dtype == "f32":
                    x, h, r = ctx.bicgstab(b.astype(np.float32).astype(np.float64), tol=1e-5)
                    bars_f32(x, h, r, xo, ho, ro)
                else:
                    x, h, r = ctx.bicgstab(b, tol=1e-10)
                    bars(x, h, r, xo, ho, ro, floor=FLOOR_BS)
                    assert r.half_step_exit == ro.half_step_exit
                    ctx.set_option("poll_batch", 3)
                    x2, h2, r2 = ctx.bicgstab(b, tol=1e-10)
                    assert r2.iterations == r.iterations and np.array_equal(x2, x) and np.array_equal(h2, h)
                    x0 = np.random.default_rng(n).standard_normal(n)
                    xo5, ho5, ro5 = oracle.bicgstab(A, b, x0=x0, tol=1e-30, maxit=5)
                    x5, h5, r5 = ctx.bicgstab(b, x0=x0, tol=1e-30, maxit=5)
                    assert r5.status == ks.KS_EMAXIT and r5.iterations == 5 and len(h5) == 5
                    bars(x5, h5, r5, xo5, ho5, ro5, iters_tol=0, floor=FLOOR_BS)
                its.append(r.iterations)
        assert abs(its[0] - its[1]) <= 2


@pytest.mark.parametrize("lay", layouts())
def test_multi_bicgstab(lay):
    P = need(lay)
    for n, kd in [(1024, 4), (4096, 16), (1001, 4)]:
        A, b = synth.gdd(n, kd)
        xo, ho, ro = oracle.bicgstab(A, b, tol=1e-10)
        with context(n, lay) as ctx:
            ctx.generate("dd", seed=synth.SEED, kd=kd, want_b=False)
            x, h, r = ctx.bicgstab(b, tol=1e-10)
        bars(x, h, r, xo, ho, ro, floor=FLOOR_BS)
        assert r.half_step_exit == ro.half_step_exit


@pytest.mark.parametrize("lay", layouts(shared=()))
def test_fused_collectives_bitwise_equal_nccl(lay):
    """NEXT-1: the fused NVLink peer-store collectives carry the same partials and
    sum them in the same rank order as the NCCL allgathers, so x, the history and
    the iteration count must be bitwise identical in both modes (and with graphs)."""
    P = need(lay)
    n = 4100
    D, bd = synth.gdd(n, 16)
    Cs, cs, bs = synth.gspd(4096, 1e4)
    with context(n, lay) as ctx, context(4096, lay) as cc:
        ctx.generate("dd", seed=synth.SEED, kd=16, want_b=False)
        cc.generate("spd", seed=synth.SEED, table=cs, want_b=False)
        assert ctx.get_option("fused_comm") == 1, "peer access expected on NVSwitch B200s"
        res = {}
        for fused, graphs in [(0, 0), (1, 0), (1, 1)]:
            for cx in (ctx, cc):
                cx.set_option("fused_comm", fused)
                cx.set_option("use_graphs", graphs)
                cx.set_option("persistent", 0)
            res[(fused, graphs)] = (ctx.bicgstab(bd, tol=1e-10), cc.cg(bs, tol=1e-10),
                                    ctx.bicgstab(bd, tol=0.0, maxit=37))
        ref = res[(0, 0)]
        for key, val in res.items():
            for (x, h, r), (xr, hr, rr) in zip(val, ref):
                assert r.iterations == rr.iterations, key
                assert np.array_equal(x, xr) and np.array_equal(h, hr), key
    xo, ho, ro = oracle.bicgstab(D, bd, tol=1e-10)
    x, h, r = ref[0]
    bars(x, h, r, xo, ho, ro, floor=FLOOR_BS)
    xo, ho, ro = oracle.cg(Cs, bs, tol=1e-10)
    x, h, r = ref[1]
    bars(x, h, r, xo, ho, ro)


@pytest.mark.parametrize("lay", layouts(shared=()))
def test_multi_persistent_fused(lay):
    """NEXT-1 + NEXT-2 together: persistent cooperative kernels on every GPU with
    the fused NVLink exchange; bars vs the oracle; identical on repeat."""
    P = need(lay)
    D, bd = synth.gdd(4096, 16)
    Cs, cs, bs = synth.gspd(4096, 1e4)
    with context(4096, lay) as ctx, context(4096, lay) as cc:
        ctx.generate("dd", seed=synth.SEED, kd=16, want_b=False)
        cc.generate("spd", seed=synth.SEED, table=cs, want_b=False)
        for cx in (ctx, cc):
            cx.set_option("persistent", 1)
            assert cx.get_option("persistent") == 1
        x, h, r = ctx.bicgstab(bd, tol=1e-10)
        x2, h2, r2 = ctx.bicgstab(bd, tol=1e-10)
        xc, hc, rc = cc.cg(bs, tol=1e-10)
    assert np.array_equal(x, x2) and np.array_equal(h, h2)
    xo, ho, ro = oracle.bicgstab(D, bd, tol=1e-10)
    bars(x, h, r, xo, ho, ro, floor=FLOOR_BS)
    xo, ho, ro = oracle.cg(Cs, bs, tol=1e-10)
    bars(xc, hc, rc, xo, ho, ro)


@pytest.mark.parametrize("lay", layouts(gpus=(), shared=(2, 4)))
def test_emulated_ranks_persistent_one_gpu(lay):
    """P ranks on ONE GPU run the fused persistent kernels (A4 / B2 over the fused
    exchange, NEXT-1) as ONE cooperative launch over all ranks' CTAs (rank = block /
    g): the CTAs that wait on each other's LL words / flags are co-resident by
    construction.  CG and BiCGSTAB vs the oracle, a fixed-length BiCGSTAB (k_end's
    last-step test), LL vs flag handovers bitwise equal, jitter at every sync point
    bitwise equal, and the launch count of one emulated launch per solve."""
    P = need(lay)
    n = 4100
    D, bd = synth.gdd(n, 16)
    Cs, cs, bs = synth.gspd(4096, 1e4)
    with context(n, lay) as ctx, context(4096, lay) as cc:
        ctx.generate("dd", seed=synth.SEED, kd=16, want_b=False)
        cc.generate("spd", seed=synth.SEED, table=cs, want_b=False)
        res = {}
        for ll, jit in ((1, 0), (0, 0), (1, 7), (0, 0x9E3779B1)):
            for cx in (ctx, cc):
                cx.set_option("ll_xchg", ll)
                cx.set_option("jitter", jit)
            res[(ll, jit)] = (ctx.bicgstab(bd, tol=1e-10), cc.cg(bs, tol=1e-10),
                              ctx.bicgstab(bd, tol=0.0, maxit=9))
        ref = res[(1, 0)]
        for key, val in res.items():
            for (x, h, r), (xr, hr, rr) in zip(val, ref):
                assert r.iterations == rr.iterations and r.status == rr.status, key
                assert np.array_equal(x, xr) and np.array_equal(h, hr), key
        for _, _, r in ref:
            assert r.kernel_launches <= 8, r.kernel_launches      # one emulated launch per solve
    xo, ho, ro = oracle.bicgstab(D, bd, tol=1e-10)
    x, h, r = ref[0]
    bars(x, h, r, xo, ho, ro, floor=FLOOR_BS)
    xo, ho, ro = oracle.cg(Cs, bs, tol=1e-10)
    x, h, r = ref[1]
    bars(x, h, r, xo, ho, ro)
    xo, ho, ro = oracle.bicgstab(D, bd, tol=0.0, maxit=9)
    x, h, r = ref[2]
    assert r.status == ks.KS_EMAXIT and r.iterations == 9
    bars(x, h, r, xo, ho, ro, iters_tol=0, floor=FLOOR_BS)


@pytest.mark.parametrize("lay", layouts(shared=()))
def test_ll_handovers_bitwise_equal_flags(lay):
    """KS_OPT_LL_XCHG: the persistent kernels over P GPUs hand the r / v slices and the
    rank partials over as LL words (no fence, no flag) instead of stores + fence + epoch
    flag; the same values are summed in the same order, so x, the history and the
    iteration count must be bitwise identical in both modes -- single- and multi-launch
    (poll batch), x0, fixed length (the last step's test in k_end), CG and BiCGSTAB --
    and meet the bars vs the oracle."""
    P = need(lay)
    n = 4100
    D, bd = synth.gdd(n, 16)
    Cs, cs, bs = synth.gspd(4096, 1e4)
    x0 = np.random.default_rng(P).standard_normal(n)
    with context(n, lay) as ctx, context(4096, lay) as cc:
        ctx.generate("dd", seed=synth.SEED, kd=16, want_b=False)
        cc.generate("spd", seed=synth.SEED, table=cs, want_b=False)
        res = {}
        for ll in (0, 1):
            for batch in (0, 5):
                for cx in (ctx, cc):
                    cx.set_option("persistent", 1)
                    cx.set_option("small", 0)
                    cx.set_option("ll_xchg", ll)
                    cx.set_option("poll_batch", batch)
                    assert cx.get_option("ll_xchg") == ll
                res[(ll, batch)] = (ctx.bicgstab(bd, tol=1e-10), cc.cg(bs, tol=1e-10),
                                    ctx.bicgstab(bd, x0=x0, tol=0.0, maxit=13),
                                    cc.cg(bs, x0=x0[:4096], tol=0.0, maxit=17))
        ref = res[(0, 0)]
        for key, val in res.items():
            for (x, h, r), (xr, hr, rr) in zip(val, ref):
                assert r.iterations == rr.iterations and r.status == rr.status, key
                assert np.array_equal(x, xr) and np.array_equal(h, hr), key
    xo, ho, ro = oracle.bicgstab(D, bd, tol=1e-10)
    x, h, r = ref[0]
    bars(x, h, r, xo, ho, ro, floor=FLOOR_BS)
    xo, ho, ro = oracle.cg(Cs, bs, tol=1e-10)
    x, h, r = ref[1]
    bars(x, h, r, xo, ho, ro)


@pytest.mark.parametrize("lay", layouts())
@pytest.mark.parametrize("fused", [1, 0])
def test_multi_bicg(lay, fused):
    """NEXT-3 BiCG at P GPUs: K1T partials reduce-scattered either inside K1T over
    NVLink peer stores (fused = 1, default) or by ncclReduceScatter (fused = 0; ranks
    sharing a GPU: the host-driven reduce-scatter); x0 and maxit included."""
    P = need(lay)
    if fused and lay[0] == "shared":
        pytest.skip("ranks sharing a GPU run the host-driven collectives only")
    for n, kd in [(1024, 4), (4099, 16)]:
        A, b = synth.gdd(n, kd)
        xo, ho, ro = oracle.bicg(A, b, tol=1e-10)
        with context(n, lay) as ctx:
            ctx.set_option("fused_comm", fused)
            assert ctx.get_option("fused_comm") == fused
            ctx.generate("dd", seed=synth.SEED, kd=kd, want_b=False)
            x, h, r = ctx.bicg(b, tol=1e-10)
            xt = np.random.default_rng(3).standard_normal(n)
            yt = ctx.matvec_t(xt)
            x0 = np.random.default_rng(5).standard_normal(n)
            xo5, ho5, ro5 = oracle.bicg(A, b, x0=x0, tol=1e-30, maxit=5)
            x5, h5, r5 = ctx.bicg(b, x0=x0, tol=1e-30, maxit=5)
            assert r5.status == ks.KS_EMAXIT and r5.iterations == 5
            bars(x5, h5, r5, xo5, ho5, ro5, iters_tol=0)
        bars(x, h, r, xo, ho, ro)
        gemv_bound_check(np.ascontiguousarray(A.T), xt, yt)


@pytest.mark.parametrize("lay", layouts())
@pytest.mark.parametrize("persistent", [0, 1])
def test_multi_gmres(lay, persistent):
    """NEXT-3 GMRES(m) at P GPUs: multi-kernel path with NCCL exchanges of the CGS2
    partial dots (persistent = 0), or one persistent kernel per restart cycle with
    the exchanges fused over NVLink (persistent = 1); x0, maxit and a restart
    length that does not divide maxit included."""
    P = need(lay)
    for n, kd, m in [(1024, 16, 30), (4099, 16, 8), (2050, 4, 3)]:
        A, b = synth.gdd(n, kd)
        x0 = np.random.default_rng(n).standard_normal(n) if n == 2050 else None
        xo, ho, ro = oracle.gmres(A, b, x0=x0, tol=1e-10, restart=m)
        with context(n, lay) as ctx:
            ctx.set_option("persistent", persistent)
            ctx.generate("dd", seed=synth.SEED, kd=kd, want_b=False)
            fused = 0 if lay[0] == "shared" else 1       # shared GPU: host collectives, multi-kernel
            assert ctx.get_option("persistent") == (persistent and fused) and ctx.get_option("fused_comm") == fused
            x, h, r = ctx.gmres(b, x0=x0, tol=1e-10, restart=m)
            bars(x, h, r, xo, ho, ro)
            xo7, ho7, ro7 = oracle.gmres(A, b, x0=x0, tol=1e-30, restart=m, maxit=7)
            x7, h7, r7 = ctx.gmres(b, x0=x0, tol=1e-30, restart=m, maxit=7)
            assert r7.status == ks.KS_EMAXIT and r7.iterations == 7
            bars(x7, h7, r7, xo7, ho7, ro7, iters_tol=0)


@pytest.mark.parametrize("lay", layouts(shared=()))
def test_multi_f32(lay):
    """NEXT-4 at P GPUs: FP32 persistent kernels with the fused NVLink exchange."""
    P = need(lay)
    from test_gpu_parity import bars_f32
    n = 4096
    A, b = synth.gdd(n, 16)
    xo, ho, ro = oracle.bicgstab_f32(A, b, tol=1e-5)
    Cs, cs, bs = synth.gspd(n, 1e2)
    xc, hc, rc = oracle.cg_f32(Cs, bs, tol=1e-5)
    with context(n, lay, dtype="f32") as ctx, context(n, lay, dtype="f32") as cc:
        ctx.generate("dd", seed=synth.SEED, kd=16, want_b=False)
        cc.generate("spd", seed=synth.SEED, table=cs, want_b=False)
        x, h, r = ctx.bicgstab(b.astype(np.float32).astype(np.float64), tol=1e-5)
        x2, h2, r2 = cc.cg(bs.astype(np.float32).astype(np.float64), tol=1e-5)
    bars_f32(x, h, r, xo, ho, ro)
    bars_f32(x2, h2, r2, xc, hc, rc)


@pytest.mark.parametrize("lay", layouts(gpus=(2,), shared=(2,)))
def test_multi_edge_cases(lay):
    need(lay)
    n = 64
    A = synth.random_spd(n, 10.0, 1)
    with context(n, lay) as ctx:
        ctx.load_rows(A)
        x, h, r = ctx.cg(np.zeros(n), tol=1e-10)
        assert r.iterations == 0 and np.all(x == 0)
        b = np.random.default_rng(0).standard_normal(n)
        x, h, r = ctx.cg(b, tol=1e-30, maxit=5)
        assert r.status == ks.KS_EMAXIT and r.iterations == 5
        x0 = np.random.default_rng(1).standard_normal(n)
        xo, ho, ro = oracle.cg(A, b, x0=x0, tol=1e-10)
        x, h, r = ctx.cg(b, x0=x0, tol=1e-10)
        bars(x, h, r, xo, ho, ro)


@pytest.mark.parametrize("lay", layouts(gpus=(2,), shared=(2,)))
def test_partial_load_is_an_error_on_every_rank(lay):
    """Single process driving 2 GPUs with only the first shard loaded: every call
    that runs a collective schedule returns KS_ESTATE up front (no rank enters a
    fused exchange its peer never joins), and the context stays usable."""
    need(lay)
    n = 512
    A = synth.random_spd(n, 10.0, 3)
    b = np.random.default_rng(3).standard_normal(n)
    with context(n, lay) as ctx:
        r0, r1 = ctx.row_range(0)
        ctx.load_rows(A[r0:r1], r0)
        for call in (lambda: ctx.cg(b), lambda: ctx.bicgstab(b), lambda: ctx.bicg(b),
                     lambda: ctx.gmres(b), lambda: ctx.matvec(b), lambda: ctx.matvec_t(b)):
            with pytest.raises(ks.KsError) as e:
                call()
            assert e.value.status == ks.KS_ESTATE
        ctx.load_rows(A[r1:], r1)
        xo, ho, ro = oracle.cg(A, b, tol=1e-10)
        x, h, r = ctx.cg(b, tol=1e-10)
        bars(x, h, r, xo, ho, ro)


def _skew_run(tmp_path, delay, tmo, port):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.join(ROOT, "tools", "dist_skew.py"), "1024", str(delay), str(tmo), str(tmp_path)]
    subprocess.run(cmd, check=True, timeout=300, cwd=ROOT)
    return [json.load(open(tmp_path / f"skew_r{g}.json")) for g in range(2)]


@needs2
def test_solve_start_rendezvous_absorbs_host_skew(tmp_path):
    """One process per GPU, the last rank calls every solve 12 s after its peer --
    beyond the 10 s bound of the in-loop waits.  The on-device rendezvous at solve
    start (k_join, default bound 120 s) absorbs it: both ranks converge with
    identical results."""
    res = _skew_run(tmp_path, 12.0, 120000, 29561)
    for name in ("cg", "bicgstab"):
        assert res[0][name]["status"] == ks.KS_OK and res[1][name]["status"] == ks.KS_OK, res
        assert res[0][name] == res[1][name]


@needs2
def test_solve_start_rendezvous_times_out_without_hanging(tmp_path):
    """Join bound 2 s, peer 6 s late: the early rank fails with KS_ENCCL and the late
    rank (which finds the early rank's join flag, then waits in the loop for
    exchanges that never come) fails too -- an error on both, never a hang."""
    res = _skew_run(tmp_path, 6.0, 2000, 29563)
    assert res[0]["cg"]["status"] == ks.KS_ENCCL, res
    assert res[1]["cg"]["status"] == ks.KS_ENCCL, res


@needs2
@pytest.mark.parametrize("P", PS)
def test_torchrun_borrowed_comm(tmp_path, P):
    """One process per GPU (torchrun, nccl); every rank returns the same x and
    history; results meet the bars vs the oracle."""
    if ngpu() < P:
        pytest.skip(f"needs {P} GPUs")
    n = 4096
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={P}",
           "--master-addr=127.0.0.1", f"--master-port={29500 + P}",
           os.path.join(ROOT, "tools", "dist_solve.py"), str(n), str(tmp_path)]
    subprocess.run(cmd, check=True, timeout=600, cwd=ROOT)
    res = [json.load(open(tmp_path / f"dist_{n}_r{g}.json")) for g in range(P)]
    for key in ("cg", "bs"):
        for g in range(1, P):
            assert res[g][key]["x"] == res[0][key]["x"], key     # bitwise identical on all ranks
            assert res[g][key]["h"] == res[0][key]["h"], key
            assert res[g][key]["it"] == res[0][key]["it"], key
    As, c, b = synth.gspd(n, 1e4)
    xo, ho, ro = oracle.cg(As, b, tol=1e-10)
    R = res[0]["cg"]

    class Rep:
        iterations = R["it"]
    bars(np.array(R["x"]), np.array(R["h"]), Rep, xo, ho, ro)
    assert res[0]["fused_effective"] == 1 and res[0]["persistent_effective"] == 1
    assert res[0]["bs_mode1"] == res[0]["bs_mode0"]           # fused == NCCL, bitwise
    for g in range(1, P):
        assert res[g]["bs_persistent"] == res[0]["bs_persistent"]
    y = np.array(res[0]["matvec"])
    gemv_bound_check(As, b, y)
    A, b = synth.gdd(n, 16)
    xo, ho, ro = oracle.bicgstab(A, b, tol=1e-10)
    R = res[0]["bs"]
    Rep.iterations = R["it"]
    bars(np.array(R["x"]), np.array(R["h"]), Rep, xo, ho, ro, floor=FLOOR_BS)
    R = res[0]["bs_persistent"]
    Rep.iterations = R["it"]
    bars(np.array(R["x"]), np.array(R["h"]), Rep, xo, ho, ro, floor=FLOOR_BS)
    xo, ho, ro = oracle.gmres(A, b, tol=1e-10, restart=20)
    R = res[0]["gmres"]
    Rep.iterations = R["it"]
    bars(np.array(R["x"]), np.array(R["h"]), Rep, xo, ho, ro)
    for g in range(1, P):
        assert res[g]["gmres"] == res[0]["gmres"]
    A, b = synth.gdd(n, 4)
    xo, ho, ro = oracle.bicgstab(A, b, tol=1e-10)
    R = res[0]["bs_loaded"]
    Rep.iterations = R["it"]
    bars(np.array(R["x"]), np.array(R["h"]), Rep, xo, ho, ro, floor=FLOOR_BS)


@pytest.mark.parametrize("lay", layouts(shared=(2,)))
def test_multi_fullsize_65536(lay):
    """C3/C3' at P GPUs, default path (persistent + fused): CG vs the closed form
    and the survey's counts; BiCGSTAB counts/histories and the true residual by the
    oracle with on-the-fly rows (pins P6, P11, P14 at scale).  The C3 history/x gate
    vs the oracle's full solve at every P is test_gpu_fullsize.py's."""
    P = need(lay)
    n = 65536
    c = synth.spd_table(n, 1e4)
    with context(n, lay) as ctx:
        b = ctx.generate("spd", seed=synth.SEED, table=c)
        x, h, r = ctx.cg(b, tol=1e-10)
    assert r.converged and abs(r.iterations - 840) <= 2
    assert np.allclose(h[:3], [0.5745285, 0.4442545, 0.3710058], rtol=5e-7, atol=0)
    xcf = oracle.spd_exact_solve_ld(c, synth.SEED, b)
    assert np.linalg.norm(x - xcf) <= 1e4 * 1e-10 * np.linalg.norm(xcf)
    with context(n, lay) as ctx:
        b = ctx.generate("dd", seed=synth.SEED, kd=16)
        x, h, r = ctx.bicgstab(b, tol=1e-10)
    assert r.converged and abs(r.iterations - 23) <= 2
    assert np.allclose(h[:3], [0.3187527, 0.1602609, 0.08888871], rtol=5e-7, atol=0)
    op = oracle.Operator(gen=synth.spec("dd", n, kd=16), threads=os.cpu_count() or 1)
    assert oracle.true_relres_ld(op, b, x) <= 10 * 1e-10


@pytest.mark.parametrize("lay", layouts(shared=(2,)))
def test_c4_131072_multi(lay):
    """C4 (n = 131072, 137 GB in total) strong-scaled over P GPUs: CG to tol 1e-10
    vs the closed form (P6), the survey count 979 (P14), the same count as one GPU
    would take (P13: survey App. A.8), and sampled true-residual rows by the oracle
    (P11, on-the-fly rows)."""
    P = need(lay)
    n = 131072
    c = synth.spd_table(n, 1e4)
    with context(n, lay) as ctx:
        b = ctx.generate("spd", seed=synth.SEED, table=c)
        x, h, r = ctx.cg(b, tol=1e-10)
    assert r.converged and abs(r.iterations - 979) <= 2, r
    xcf = oracle.spd_exact_solve_ld(c, synth.SEED, b)
    assert np.linalg.norm(x - xcf) <= 1e4 * 1e-10 * np.linalg.norm(xcf)
    assert r.true_relres <= 10 * 1e-10
    op = oracle.Operator(gen=synth.spec("spd", n, kappa=1e4), threads=min(8, os.cpu_count() or 1))
    nb = float(np.linalg.norm(b))
    for i in (0, 16383, 16384, 65535, 65536, 131071):
        assert abs(b[i] - op.rows(i, 1, x)[0]) <= 10 * 1e-10 * nb


@pytest.mark.parametrize("P", [4, 8])
def test_c5_262144(P):
    """C5: n = 262144 (550 GB in total; 137 / 69 GB per GPU at P = 4 / 8): CG vs the
    closed form (survey: 1070 iterations); BiCGSTAB converges with a small true
    residual checked by the oracle on sampled rows (on-the-fly generation)."""
    if ngpu() < P:
        pytest.skip(f"needs {P} GPUs (C5 does not fit fewer)")
    n = 262144
    c = synth.spd_table(n, 1e4)
    with ks.Context(n, ngpus=P) as ctx:
        b = ctx.generate("spd", seed=synth.SEED, table=c)
        x, h, r = ctx.cg(b, tol=1e-10)
        assert r.converged and abs(r.iterations - 1070) <= 2
        xcf = oracle.spd_exact_solve_ld(c, synth.SEED, b)
        assert np.linalg.norm(x - xcf) <= 1e4 * 1e-10 * np.linalg.norm(xcf)
    with ks.Context(n, ngpus=P) as ctx:
        b = ctx.generate("dd", seed=synth.SEED, kd=16)
        x, h, r = ctx.bicgstab(b, tol=1e-10)
    assert r.converged and r.iterations <= 30 and r.true_relres <= 10 * 1e-10
    op = oracle.Operator(gen=synth.spec("dd", n, kd=16), threads=min(8, os.cpu_count() or 1))
    nb = float(np.linalg.norm(b))
    for i in (0, 1, 131071, 131072, 262143):
        assert abs(b[i] - op.rows(i, 1, x)[0]) <= 10 * 1e-10 * nb
