"""Race detection by schedule perturbation (KS_OPT_JITTER).

With a jitter seed every synchronisation point of the persistent, small, tiny and
multi-RHS kernels (grid-barrier arrival and departure, flag publish and wait, LL
store and poll) makes a pseudo-random quarter of the warps sleep up to ~4 us, so
CTAs, warps and ranks reach each hand-over in a different order on every run.  The
kernels' results must not depend on that order (fixed summation trees, epoch-tagged
exchanges): x, the residual history and the iteration count
with jitter must equal the run without it BIT FOR BIT.  A missing barrier, fence or
double buffer (the round-1 launch-start race, `a6f0a97`, was one) shows up here as a
difference or a timeout.  Each case runs single-launch and multi-launch (poll batch)
solves, x0 and fixed-length runs, on one GPU and on P GPUs.
The loop time with jitter must exceed the one without: the delays really ran."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu
ks = pytest.importorskip("paper_1511_07174_b200")

from layouts import context, need  # noqa: E402

SEEDS = (7, 0x9E3779B1)
LAYS = [pytest.param(("gpus", 1), id="gpus1"), pytest.param(("gpus", 2), id="gpus2"),
        pytest.param(("gpus", 4), id="gpus4")]


def gspd_any(n):
    """SPD with eigenvalues in [1, 1e3] for any n (the G-SPD recipe needs a power of
    two): A = Q diag Q^T from a seeded orthogonal Q."""
    rng = np.random.default_rng(n)
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    lam = np.geomspace(1.0, 1e3, n)
    return (Q * lam) @ Q.T, synth.rhs(n)


def same(a, b):
    (x, h, r), (y, g, s) = a, b
    return r.iterations == s.iterations and r.status == s.status and np.array_equal(x, y) and \
        np.array_equal(h, g)


def jitter_runs(ctx, solve):
    """solve() without jitter twice, then with every seed: all bitwise equal; the
    jittered loops take longer than the fastest plain one."""
    ctx.set_option("jitter", 0)
    ref = solve()
    again = solve()
    assert same(ref, again), "not repeatable even without jitter"
    t0 = min(ref[2].seconds_loop, again[2].seconds_loop)
    slower = 0
    for seed in SEEDS:
        ctx.set_option("jitter", seed)
        assert ctx.get_option("jitter") == seed
        out = solve()
        assert same(out, ref), f"result changed under jitter seed {seed:#x}"
        slower += out[2].seconds_loop > 1.05 * t0
    ctx.set_option("jitter", 0)
    assert slower >= 1, "jitter had no visible effect on the loop time"
    return ref


@pytest.mark.parametrize("lay", LAYS)
@pytest.mark.parametrize("path", ["persistent", "small"])
def test_race_cg_bicgstab(lay, path):
    P = need(lay)
    n = 4100 if path == "persistent" else 2003
    A, b = gspd_any(n)
    D, bd = synth.gdd(n, 4)
    x0 = np.random.default_rng(1).standard_normal(n)
    with context(n, lay) as ctx, context(n, lay) as dtx:
        for cx in (ctx, dtx):
            cx.set_option("tiny", 0)
            cx.set_option("small", 0 if path == "persistent" else 1)
            cx.set_option("persistent", 1)
        ctx.load_rows(A)
        dtx.load_rows(D)
        for batch in (0, 7):
            for cx in (ctx, dtx):
                cx.set_option("poll_batch", batch)
            jitter_runs(ctx, lambda: ctx.cg(b, tol=1e-10))
            jitter_runs(ctx, lambda: ctx.cg(b, x0=x0, tol=0.0, maxit=23))
            jitter_runs(dtx, lambda: dtx.bicgstab(bd, tol=1e-10))
            jitter_runs(dtx, lambda: dtx.bicgstab(bd, x0=x0, tol=0.0, maxit=9))
    assert P >= 1


@pytest.mark.parametrize("lay", LAYS + [pytest.param(("shared", 2), id="shared2"),
                                        pytest.param(("shared", 4), id="shared4")])
def test_race_tiny(lay):
    need(lay)
    n = 1000
    A, b = gspd_any(n)
    D, bd = synth.gdd(n, 4)
    with context(n, lay) as ctx, context(n, lay) as dtx:
        ctx.load_rows(A)
        dtx.load_rows(D)
        jitter_runs(ctx, lambda: ctx.cg(b, tol=1e-10))
        jitter_runs(dtx, lambda: dtx.bicgstab(bd, tol=1e-10))


@pytest.mark.parametrize("lay", LAYS)
def test_race_multi_rhs(lay):
    need(lay)
    n = 2050
    A, _ = gspd_any(n)
    D, _ = synth.gdd(n, 4)
    B = np.column_stack([synth.rhs(n, synth.SEED + j) for j in range(4)])
    with context(n, lay) as ctx, context(n, lay) as dtx:
        ctx.load_rows(A)
        dtx.load_rows(D)
        for cx, fn in ((ctx, ctx.cg_multi), (dtx, dtx.bicgstab_multi)):
            cx.set_option("jitter", 0)
            X, h, r = fn(B, tol=1e-10)
            t0 = max(q.seconds_loop for q in r)
            for seed in SEEDS:
                cx.set_option("jitter", seed)
                Xj, hj, rj = fn(B, tol=1e-10)
                assert np.array_equal(Xj, X), seed
                for k in range(B.shape[1]):
                    assert rj[k].iterations == r[k].iterations and np.array_equal(hj[k], h[k])
            cx.set_option("jitter", 0)
            assert t0 > 0


@pytest.mark.parametrize("lay", [pytest.param(("gpus", 1), id="gpus1"), pytest.param(("gpus", 2), id="gpus2")])
def test_race_gmres_and_f32(lay):
    need(lay)
    n = 1030
    D, bd = synth.gdd(n, 16)
    with context(n, lay) as ctx:
        ctx.set_option("persistent", 1)
        ctx.load_rows(D)
        jitter_runs(ctx, lambda: ctx.gmres(bd, tol=1e-10, restart=30))
    with context(n, lay, dtype="f32") as ctx:
        ctx.set_option("persistent", 1)
        ctx.set_option("small", 0)
        ctx.load_rows(D)
        bf = bd.astype(np.float32).astype(np.float64)
        jitter_runs(ctx, lambda: ctx.bicgstab(bf, tol=1e-5))
