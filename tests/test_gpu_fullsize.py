"""Full-size parity at BASELINE.json's headline size n = 65536 (configs C3/C3'),
in the launch configuration bench.py times (auto K1 config, one GPU, generated
inputs).  The oracle cannot run whole solves at this size in seconds, so this file
checks what it can compute one by one, and properties that hold at any size:
  * sampled GEMV rows vs the oracle's on-the-fly generated rows (P9 bound),
  * CG x vs the long-double closed-form solution (P6), survey App. A.8 counts (P14),
  * BiCGSTAB true residual by the oracle with on-the-fly rows (P11),
  * the C3 gate: the WHOLE BiCGSTAB history (23 iterations)
    and x vs the oracle's own full solve on G-DD(65536, 16) -- the oracle stores
    the 34 GB matrix on the host when RAM allows (else generates rows on the fly)
    and runs row-parallel on all host cores (every row sum sequential, so bitwise
    the 1-thread oracle) -- on 1 GPU and on every P in {2, 4, 8} the box has.
"""
import os

import numpy as np
import pytest

import oracle
import synth

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
ks = pytest.importorskip("paper_1511_07174_b200")

from test_gpu_parity import FLOOR_BS, bars, gamma  # noqa: E402

N = 65536
THREADS = os.cpu_count() or 1
from layouts import context, layouts, need  # noqa: E402


def _mem_available() -> int:
    try:
        with open("/proc/meminfo") as f:
            for ln in f:
                if ln.startswith("MemAvailable:"):
                    return int(ln.split()[1]) * 1024
    except OSError:
        pass
    return 0


def oracle_operator(kind: str, n: int, **kw):
    """The oracle's operator for a generated matrix at full size: stored rows
    (expanded by the oracle's own generator on all host cores) when the host has
    room for them, else rows generated on the fly.  Same entries, same order,
    bitwise the same GEMV either way (test_true_relres_stored_equals_on_the_fly)."""
    spec = synth.spec(kind, n, **kw)
    if _mem_available() > 1.25 * 8.0 * n * n + 16e9:
        A = oracle.gen_rows(spec, 0, n, threads=THREADS)
        return oracle.Operator(A, threads=THREADS), "stored"
    return oracle.Operator(gen=spec, threads=THREADS), "on-the-fly"


def _ngpu():
    import torch
    return torch.cuda.device_count()


@pytest.fixture(scope="module")
def c3_oracle():
    """The oracle's full C3 solve: BiCGSTAB on G-DD(65536, 16), tol 1e-10, x0 = 0
    (46 GEMVs).  Survey App. A.8: 23 iterations, full-step exit."""
    b = synth.rhs(N)
    op, mode = oracle_operator("dd", N, kd=16)
    xo, ho, ro = oracle.bicgstab(op, b, tol=1e-10)
    del op
    return b, xo, ho, ro, mode


SAMPLE =[0, 1, 511, 512, 4095, 32767, 32768, 65534, 65535] + \
    list(np.random.default_rng(65536).integers(0, N, 23))


def _rows_check(spec, x, y):
    op = oracle.Operator(gen=spec, threads=min(THREADS, 8))
    for i in SAMPLE:
        yo = op.rows(int(i), 1, x)[0]
        a = oracle.gen_rows(spec, int(i), 1)[0]
        bound = 2 * gamma(N) * float(np.abs(a) @ np.abs(x))
        assert abs(y[i] - yo) <= bound, (i, y[i], yo, bound)


def test_fullsize_gemv_sampled_rows():
    x = synth.rhs(N, synth.SEED2)
    for kind in ("dd", "spd"):
        spec = synth.spec(kind, N, kappa=1e4, kd=16)
        with ks.Context(N) as ctx:
            ctx.generate(kind, seed=synth.SEED, table=spec["table"], kd=16, want_b=False)
            y = ctx.matvec(x)
        _rows_check(spec, x, y)


def test_fullsize_cg_closed_form():
    """C3': G-SPD(65536, 1e4), tol 1e-10: x vs the closed form, counts/histories vs
    the survey's independent spec implementation (reference values)."""
    c = synth.spd_table(N, 1e4)
    with ks.Context(N) as ctx:
        b = ctx.generate("spd", seed=synth.SEED, table=c)
        x, h, r = ctx.cg(b, tol=1e-10)
    assert r.converged and abs(r.iterations - 840) <= 2, r
    assert np.allclose(h[:3], [0.5745285, 0.4442545, 0.3710058], rtol=5e-7, atol=0)
    xcf = oracle.spd_exact_solve_ld(c, synth.SEED, b)
    assert np.linalg.norm(x - xcf) <= 1e4 * 1e-10 * np.linalg.norm(xcf)
    assert r.true_relres <= 10 * 1e-10
    # sampled true residual entries by the oracle (on-the-fly rows)
    spec = synth.spec("spd", N, kappa=1e4)
    op = oracle.Operator(gen=spec, threads=min(THREADS, 8))
    nb = float(np.linalg.norm(b))
    for i in SAMPLE[:12]:
        ri = b[i] - op.rows(int(i), 1, x)[0]
        assert abs(ri) <= 10 * 1e-10 * nb


def test_fullsize_bicgstab_true_residual_and_first_iterations():
    """C3: G-DD(65536, 16), tol 1e-10."""
    spec = synth.spec("dd", N, kd=16)
    with ks.Context(N) as ctx:
        b = ctx.generate("dd", seed=synth.SEED, kd=16)
        x, h, r = ctx.bicgstab(b, tol=1e-10)
        x2, h2, r2 = ctx.bicgstab(b, tol=0.0, maxit=2)       # bench mode, fixed length
    assert r.converged and abs(r.iterations - 23) <= 2, r
    assert np.allclose(h[:3], [0.3187527, 0.1602609, 0.08888871], rtol=5e-7, atol=0)
    op = oracle.Operator(gen=spec, threads=THREADS)
    tr = oracle.true_relres_ld(op, b, x)
    assert tr <= 10 * 1e-10
    assert abs(tr - r.true_relres) <= 1e-3 * tr + 1e-15
    # the oracle itself, 2 iterations (4 GEMVs with on-the-fly rows)
    xo, ho, ro = oracle.bicgstab(op, b, tol=0.0, maxit=2)
    bars(x2, h2, r2, xo, ho, ro, iters_tol=0, floor=FLOOR_BS)


@pytest.mark.parametrize("lay", [pytest.param(("gpus", 1), id="gpus1")] + layouts(shared=(2,)))
def test_c3_bicgstab_full_history_and_x_vs_oracle(lay, c3_oracle):
    """C3 gate, north-star bars on the whole run at the headline size, in the
    bench's launch configuration (persistent kernels, fused exchange for P > 1):
    every history entry (Q17 floor), x within 1e-9 of the oracle's x, iteration
    count within 2 (expected: equal), same exit kind."""
    P = need(lay)
    b, xo, ho, ro, mode = c3_oracle
    assert ro.converged and ro.iterations == 23 and not ro.half_step_exit, (ro, mode)
    with context(N, lay) as ctx:
        bg = ctx.generate("dd", seed=synth.SEED, kd=16)
        assert np.array_equal(bg, b)                               # P12
        x, h, r = ctx.bicgstab(bg, tol=1e-10)
    assert r.converged and r.half_step_exit == ro.half_step_exit
    assert len(h) == r.iterations and len(ho) == ro.iterations
    bars(x, h, r, xo, ho, ro, floor=FLOOR_BS)
    k = min(len(h), len(ho))
    assert k >= 21
    assert np.all(np.abs(h[:k] - ho[:k]) <= 1e-8 * ho[:k] + FLOOR_BS)
    assert np.linalg.norm(x - xo) <= 1e-9 * np.linalg.norm(xo)


def _first50(h, ho, floor):
    k = min(50, len(h), len(ho))
    assert k == 50
    d = np.abs(h[:k] - ho[:k])
    assert np.all(d <= 1e-8 * ho[:k] + floor), float(np.max(d / ho[:k]))


@pytest.mark.parametrize("n,iters", [(32768, 623), (65536, 840)])
def test_cg_first_50_history_vs_oracle(n, iters):
    """C2 / C3': the GPU's first 50 CG residuals at tol 1e-10
    vs the oracle's own first 50 iterations (on-the-fly rows, all host cores), and
    the expected iteration count."""
    c = synth.spd_table(n, 1e4)
    with ks.Context(n) as ctx:
        b = ctx.generate("spd", seed=synth.SEED, table=c)
        x, h, r = ctx.cg(b, tol=1e-10)
    assert r.converged and abs(r.iterations - iters) <= 2, r
    op = oracle.Operator(gen=synth.spec("spd", n, kappa=1e4), threads=THREADS)
    xo, ho, ro = oracle.cg(op, b, tol=0.0, maxit=50)
    _first50(h, ho, 1e-14)


def test_c4_131072_one_gpu():
    """C4 at P = 1, the largest single-GPU config (137.4 GB of A in one B200's HBM):
    CG to tol 1e-10 vs the closed-form solution (P6), the survey's count (P14) and
    sampled true-residual entries by the oracle (P11)."""
    n = 131072
    c = synth.spd_table(n, 1e4)
    with ks.Context(n) as ctx:
        b = ctx.generate("spd", seed=synth.SEED, table=c)
        x, h, r = ctx.cg(b, tol=1e-10)
    assert r.converged and abs(r.iterations - 979) <= 2, r
    xcf = oracle.spd_exact_solve_ld(c, synth.SEED, b)
    assert np.linalg.norm(x - xcf) <= 1e4 * 1e-10 * np.linalg.norm(xcf)
    assert r.true_relres <= 10 * 1e-10
    op = oracle.Operator(gen=synth.spec("spd", n, kappa=1e4), threads=min(THREADS, 8))
    nb = float(np.linalg.norm(b))
    for i in [0, 1, 65535, 65536, 131071]:
        assert abs(b[i] - op.rows(i, 1, x)[0]) <= 10 * 1e-10 * nb


@pytest.mark.parametrize("method", ["bicg", "gmres"])
def test_fullsize_next3_true_residual(method):
    """NEXT-3 at the headline size (C3: G-DD(65536, 16), tol 1e-10) in the launch
    configuration of the defaults (BiCG: K1 + K1T; GMRES(30): persistent cycle
    kernel): converged, and the true residual recomputed by the oracle with
    on-the-fly rows (long double) within 10 tol and equal to the library's own."""
    spec = synth.spec("dd", N, kd=16)
    with ks.Context(N) as ctx:
        b = ctx.generate("dd", seed=synth.SEED, kd=16)
        kw = {"restart": 30} if method == "gmres" else {}
        x, h, r = getattr(ctx, method)(b, tol=1e-10, **kw)
    assert r.converged and r.status == ks.KS_OK and 0 < r.iterations < 200
    op = oracle.Operator(gen=spec, threads=THREADS)
    tr = oracle.true_relres_ld(op, b, x)
    assert tr <= 10 * 1e-10
    assert abs(tr - r.true_relres) <= 1e-3 * tr + 1e-15
    if method == "gmres":                      # minimal residual: non-increasing history
        assert np.all(h[1:] <= h[:-1] * (1 + 1e-12))
