"""GPU parity of multi-RHS CG (ks_cg_multi: one TMA-fed skinny GEMM per iteration,
K independent CG recurrences; reading Q30) vs the oracle, column by
column, at the north-star bars (Q17-Q19).  Inputs: G-SPD (SURVEY.md sec.8(d).2,
parity-safe: uniform spectrum), K right-hand sides from the sec.8(d).2 hash with
seeds SEED + k; ragged n (partial 32-row bands, padded 128-column chunks); nrhs
1..8 (kernel widths 4 and 8 with padding columns); every per-column exit."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu
ks = pytest.importorskip("paper_1511_07174_b200")

from test_gpu_parity import bars  # noqa: E402
from layouts import context, layouts, need  # noqa: E402


def gspd_any(n, kappa=1e3):
    A1, _, _ = synth.gspd(n + n % 2, kappa)
    return np.ascontiguousarray(A1[:n, :n])


def rhs_block(n, k):
    return np.column_stack([synth.rhs(n, synth.SEED + j) for j in range(k)])


@pytest.mark.parametrize("n,nrhs", [(1024, 1), (1024, 4), (1000, 3), (2050, 5), (4096, 8), (777, 8)])
def test_multi_rhs_parity(n, nrhs):
    A = gspd_any(n)
    B = rhs_block(n, nrhs)
    Xo, ho, ro = oracle.cg_multi(A, B, tol=1e-10)
    with ks.Context(n) as ctx:
        ctx.load_rows(A)
        X, h, r = ctx.cg_multi(B, tol=1e-10)
    for k in range(nrhs):
        bars(X[:, k], h[k], r[k], Xo[:, k], ho[k], ro[k])
        assert r[k].converged and r[k].status == ks.KS_OK


def test_multi_rhs_matches_single_rhs_cg():
    """Column k of the block solve meets the bars against the single-RHS GPU CG
    (the same recurrence through K1/the persistent kernels); single- and multi-RHS
    solves interleave on one context (their device states are independent)."""
    n = 2048
    A = gspd_any(n, 1e4)
    B = rhs_block(n, 6)
    with ks.Context(n) as ctx:
        ctx.load_rows(A)
        X, h, r = ctx.cg_multi(B, tol=1e-10)
        for k in range(6):
            x1, h1, r1 = ctx.cg(B[:, k], tol=1e-10)
            bars(X[:, k], h[k], r[k], x1, h1, r1)
        X2, h2, r2 = ctx.cg_multi(B, tol=1e-10)        # after single-RHS solves
        assert np.array_equal(X2, X) and [q.iterations for q in r2] == [q.iterations for q in r]
        X3, _, r3 = ctx.cg_multi(B, tol=0.0, maxit=7)
        assert all(q.iterations == 7 and q.status == ks.KS_EMAXIT for q in r3)


def test_multi_rhs_x0_and_exits():
    n = 600
    A = gspd_any(n)
    B = rhs_block(n, 5)
    B[:, 2] = 0.0                                    # Q6: b = 0 -> x = 0, 0 iterations
    X0 = np.random.default_rng(3).standard_normal((n, 5))
    X0[:, 4] = np.linalg.solve(A, B[:, 4])           # (near) exact start: 0-iteration exit
    Xo, ho, ro = oracle.cg_multi(A, B, X0=X0, tol=1e-10)
    with ks.Context(n) as ctx:
        ctx.load_rows(A)
        X, h, r = ctx.cg_multi(B, X0=X0, tol=1e-10)
        for k in (0, 1, 3):
            bars(X[:, k], h[k], r[k], Xo[:, k], ho[k], ro[k])
        assert r[2].iterations == 0 and r[2].converged and np.all(X[:, 2] == 0)
        assert r[4].iterations == ro[4].iterations == 0 and np.array_equal(X[:, 4], X0[:, 4])
        # maxit: every column stops at maxit = 6 with the oracle's x after 6 steps
        Xo6, ho6, _ = oracle.cg_multi(A, B[:, :2], tol=0.0, maxit=6)
        X6, h6, r6 = ctx.cg_multi(B[:, :2], tol=0.0, maxit=6)
        for k in range(2):
            assert r6[k].status == ks.KS_EMAXIT and r6[k].iterations == 6 and len(h6[k]) == 6
            assert np.linalg.norm(X6[:, k] - Xo6[:, k]) <= 1e-12 * np.linalg.norm(Xo6[:, k])
        # repeated solve: bitwise identical
        X2, h2, r2 = ctx.cg_multi(B, X0=X0, tol=1e-10)
        assert np.array_equal(X2, X) and all(np.array_equal(a, b) for a, b in zip(h, h2))


def test_multi_rhs_per_column_notspd():
    """diag(1..m, -1..-m): a right-hand side in the positive eigenspace converges, one
    touching the negative eigenspace meets <p, A p> < 0 (NOTSPD for that column only,
    x = x0); the call returns KS_ENOTSPD (worst column)."""
    m = 300
    d = np.concatenate([np.arange(1, m + 1), -np.arange(1, m + 1)]).astype(np.float64)
    A = np.diag(d)
    n = 2 * m
    b0 = np.concatenate([np.ones(m), np.zeros(m)])
    b1 = np.concatenate([np.zeros(m), np.ones(m)])
    B = np.column_stack([b0, b1])
    Xo, ho, ro = oracle.cg_multi(A, B, tol=1e-10)
    with ks.Context(n) as ctx:
        ctx.load_rows(A)
        X, h, r = ctx.cg_multi(B, tol=1e-10)
    assert ro[0].status == ks.KS_OK and r[0].status == ks.KS_OK
    bars(X[:, 0], h[0], r[0], Xo[:, 0], ho[0], ro[0])
    assert ro[1].status == r[1].status == ks.KS_ENOTSPD and r[1].iterations == ro[1].iterations == 0
    assert np.all(X[:, 1] == 0)


def test_multi_rhs_argument_errors():
    n = 64
    with ks.Context(n) as ctx:
        ctx.load_rows(np.eye(n))
        with pytest.raises(ks.KsError) as e:
            ctx.cg_multi(np.ones((n, 9)))
        assert e.value.status == ks.KS_EARG
        X, h, r = ctx.cg_multi(np.ones((n, 2)), tol=1e-12)     # A = I: 1 iteration, x = b
        assert all(q.iterations == 1 for q in r) and np.allclose(X, 1.0, rtol=0, atol=1e-15)


def _ngpu():
    import torch
    return torch.cuda.device_count()


@pytest.mark.parametrize("lay", layouts(shared=()))
def test_multi_rhs_over_p_gpus(lay):
    """Multi-RHS CG over P GPUs (row blocks; per iteration the K columns' sigma and
    rho' partials are all-reduced and the r slices gathered through the fused NVLink
    exchange inside the persistent kernel; x gathered in-kernel): per-column bars vs
    the oracle on a ragged n, with x0 and a b = 0 column; bitwise equal to a repeat."""
    P = need(lay)
    n = 2050
    A = gspd_any(n)
    B = rhs_block(n, 6)
    B[:, 3] = 0.0
    X0 = np.random.default_rng(P).standard_normal((n, 6))
    Xo, ho, ro = oracle.cg_multi(A, B, X0=X0, tol=1e-10)
    with context(n, lay) as ctx:
        assert ctx.get_option("fused_comm") == 1
        ctx.load_rows(A)
        X, h, r = ctx.cg_multi(B, X0=X0, tol=1e-10)
        for k in (0, 1, 2, 4, 5):
            bars(X[:, k], h[k], r[k], Xo[:, k], ho[k], ro[k])
        assert r[3].iterations == 0 and np.all(X[:, 3] == 0)
        X2, h2, r2 = ctx.cg_multi(B, X0=X0, tol=1e-10)
        assert np.array_equal(X2, X)
        Xs, hs, rs = ctx.cg_multi(B[:, :2], tol=0.0, maxit=5)       # fixed length, no x0
        Xso, hso, _ = oracle.cg_multi(A, B[:, :2], tol=0.0, maxit=5)
        for k in range(2):
            assert rs[k].iterations == 5
            assert np.linalg.norm(Xs[:, k] - Xso[:, k]) <= 1e-12 * np.linalg.norm(Xso[:, k])


# ---------------------------------------------------------------- multi-RHS BiCGSTAB

def gdd_block(n, k, kd=4):
    D, b = synth.gdd(n, kd)
    return D, np.column_stack([b] + [synth.rhs(n, synth.SEED + j) for j in range(1, k)])


@pytest.mark.parametrize("n,nrhs", [(1024, 1), (1000, 3), (2050, 5), (4096, 8), (777, 8)])
def test_bicgstab_multi_parity(n, nrhs):
    """Multi-RHS BiCGSTAB vs oracle.bicgstab_multi column by column (G-DD kd = 4:
    the parity-safe BiCGSTAB input), half-step exits per column."""
    from test_gpu_parity import FLOOR_BS
    D, B = gdd_block(n, nrhs)
    Xo, ho, ro = oracle.bicgstab_multi(D, B, tol=1e-10)
    with ks.Context(n) as ctx:
        ctx.load_rows(D)
        X, h, r = ctx.bicgstab_multi(B, tol=1e-10)
    for k in range(nrhs):
        bars(X[:, k], h[k], r[k], Xo[:, k], ho[k], ro[k], floor=FLOOR_BS)
        assert r[k].converged and r[k].half_step_exit == ro[k].half_step_exit
        assert r[k].matvecs == 2 * r[k].iterations - (1 if r[k].half_step_exit else 0)


def test_bicgstab_multi_exits_and_repeat():
    """x0, a b = 0 column, maxit (the oracle's x after 5 steps), a per-column
    breakdown (a rotation block), repeat bitwise, and the single-RHS GPU solver agree."""
    from test_gpu_parity import FLOOR_BS
    n = 600
    D, B = gdd_block(n, 4, kd=4)
    B[:, 2] = 0.0
    # a small x0: the history starts near 1 (the Q17 floor is in relres units; a random
    # x0 of unit size puts h_0 at ~300 and the rounding noise of the tail with it)
    X0 = 1e-3 * np.random.default_rng(5).standard_normal((n, 4))
    Xo, ho, ro = oracle.bicgstab_multi(D, B, X0=X0, tol=1e-10)
    with ks.Context(n) as ctx:
        ctx.load_rows(D)
        X, h, r = ctx.bicgstab_multi(B, X0=X0, tol=1e-10)
        for k in (0, 1, 3):
            bars(X[:, k], h[k], r[k], Xo[:, k], ho[k], ro[k], floor=FLOOR_BS)
        assert r[2].iterations == 0 and np.all(X[:, 2] == 0)
        X2, h2, r2 = ctx.bicgstab_multi(B, X0=X0, tol=1e-10)
        assert np.array_equal(X2, X)
        Xo5, _, _ = oracle.bicgstab_multi(D, B[:, :2], tol=0.0, maxit=5)
        X5, h5, r5 = ctx.bicgstab_multi(B[:, :2], tol=0.0, maxit=5)
        for k in range(2):
            assert r5[k].iterations == 5 and r5[k].status == ks.KS_EMAXIT and len(h5[k]) == 5
            assert np.linalg.norm(X5[:, k] - Xo5[:, k]) <= 1e-12 * np.linalg.norm(Xo5[:, k])
        x1, h1, r1 = ctx.bicgstab(B[:, 0], tol=1e-10)
        Xs, hs, rs = ctx.bicgstab_multi(B[:, :1], tol=1e-10)
        bars(Xs[:, 0], hs[0], rs[0], x1, h1, r1, floor=FLOOR_BS)
    A = np.zeros((n, n))
    A[: n // 2, : n // 2] = np.diag(1.0 + np.arange(n // 2) % 4)   # 4 distinct eigenvalues: a few exact steps
    for i in range(n // 2, n, 2):
        A[i, i + 1], A[i + 1, i] = 1.0, -1.0
    Bb = np.zeros((n, 2))
    Bb[: n // 2, 0] = 1.0
    Bb[n // 2, 1] = 1.0
    Xo, ho, ro = oracle.bicgstab_multi(A, Bb, tol=1e-10)
    with ks.Context(n) as ctx:
        ctx.load_rows(A)
        X, h, r = ctx.bicgstab_multi(Bb, tol=1e-10)
    assert ro[1].status == r[1].status == ks.KS_EBREAKDOWN and r[1].iterations == 0 and np.all(X[:, 1] == 0)
    assert r[0].status == ks.KS_OK
    bars(X[:, 0], h[0], r[0], Xo[:, 0], ho[0], ro[0], floor=FLOOR_BS)


@pytest.mark.parametrize("lay", layouts(shared=()))
def test_bicgstab_multi_over_p_gpus(lay):
    """Multi-RHS BiCGSTAB over P GPUs: v and r slices through every rank's exchange
    regions, the per-column dots as rank all-reduces; per-column bars vs the oracle
    (half-step exits, a b = 0 column, small x0), bitwise repeat, and the one-GPU
    result within the bars."""
    P = need(lay)
    from test_gpu_parity import FLOOR_BS
    n = 2050
    D, B = gdd_block(n, 5)
    B[:, 3] = 0.0
    X0 = 1e-3 * np.random.default_rng(P).standard_normal((n, 5))
    Xo, ho, ro = oracle.bicgstab_multi(D, B, X0=X0, tol=1e-10)
    with context(n, lay) as ctx:
        ctx.load_rows(D)
        X, h, r = ctx.bicgstab_multi(B, X0=X0, tol=1e-10)
        for k in (0, 1, 2, 4):
            bars(X[:, k], h[k], r[k], Xo[:, k], ho[k], ro[k], floor=FLOOR_BS)
            assert r[k].half_step_exit == ro[k].half_step_exit
        assert r[3].iterations == 0 and np.all(X[:, 3] == 0)
        X2, _, _ = ctx.bicgstab_multi(B, X0=X0, tol=1e-10)
        assert np.array_equal(X2, X)
