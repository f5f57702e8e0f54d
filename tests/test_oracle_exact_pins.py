"""Round-2 pins of the oracle (CPU only), each against something other than the
oracle itself:

  * or_true_relres_ld (the P11 checker, SPEC.md:563 residual contract) pinned
    TWO-SIDED: exact values it must return (x = 0 gives exactly 1; integer and
    dyadic systems whose ||b - A x|| / ||b|| is known in closed form, evaluated
    with Python's exact Fractions and a 50-digit Decimal square root), scale
    invariance, and stored == on-the-fly rows bitwise.  An upper bound alone
    would let a deflating bug (||r||/||b||^2, a dropped sqrt) pass.
  * BiCGSTAB P3 at EVERY step (PAPER.md:29 exact-arithmetic termination; SURVEY
    sec.8(c).7 P3): x_i, s_i, r_i and hist_i of the FP64 oracle vs a rational
    re-implementation of SURVEY sec.8(c).4 -- a wrong beta or omega that still
    converges changes the intermediate iterates and fails here.
  * The measurements behind DESIGN.md readings: the BiCGSTAB history floor
    (Q17: 1e-12, not 2e-13) and the two "chaotic" inputs that are not parity
    inputs (SPEC.md:560 convection-diffusion, random-sign diagonals).
"""
from decimal import Decimal, getcontext
from fractions import Fraction as F

import numpy as np
import pytest

import oracle
import synth

EPS = 2.0 ** -52


# ----------------------------------------------------- or_true_relres_ld

def _exact_ratio(A, b, x):
    """||b - A x||_2 / ||b||_2 for dyadic-rational inputs, exactly (Fractions),
    rounded once through a 50-digit Decimal square root."""
    n = len(b)
    Aq = [[F(float(v)) for v in row] for row in A]
    bq = [F(float(v)) for v in b]
    xq = [F(float(v)) for v in x]
    rr = sum((bq[i] - sum(Aq[i][j] * xq[j] for j in range(n))) ** 2 for i in range(n))
    bb = sum(v * v for v in bq)
    getcontext().prec = 50
    num = Decimal(rr.numerator) / Decimal(rr.denominator)
    den = Decimal(bb.numerator) / Decimal(bb.denominator)
    return float((num / den).sqrt())


def test_true_relres_x_zero_is_exactly_one():
    """x = 0: b - A x = b, so the ratio is exactly 1 (any A, stored or generated)."""
    rng = np.random.default_rng(11)
    for n in (1, 7, 64):
        A = rng.standard_normal((n, n))
        b = rng.standard_normal(n)
        assert oracle.true_relres_ld(A, b, np.zeros(n)) == 1.0
    for kind in ("spd", "dd"):
        op = oracle.Operator(gen=synth.spec(kind, 256, kappa=1e3, kd=16), threads=2)
        assert oracle.true_relres_ld(op, synth.rhs(256), np.zeros(256)) == 1.0


def test_true_relres_integer_closed_form():
    """Integer A, x and a chosen integer residual r*: b = A x + r*, so the exact
    value is ||r*|| / ||b||.  Perfect squares make it a short rational: r* has
    norm 13 (3,4,12) and b is built with norm^2 known exactly."""
    rng = np.random.default_rng(12)
    for trial in range(20):
        n = int(rng.integers(3, 9))
        A = rng.integers(-9, 10, (n, n)).astype(float)
        x = rng.integers(-9, 10, n).astype(float)
        r = np.zeros(n)
        r[:3] = [3.0, 4.0, 12.0]
        rng.shuffle(r)
        b = A @ x + r                                    # integers < 2^53: exact
        expect = 13.0 / float(Decimal(int(np.sum(b.astype(np.int64) ** 2))).sqrt())
        got = oracle.true_relres_ld(A, b, x)
        assert abs(got - expect) <= EPS * expect, (trial, got, expect)
    # exactly representable answers
    I4 = np.eye(4)
    x = np.array([6.0, 8.0, 0.0, 0.0])
    assert oracle.true_relres_ld(I4, x, x) == 0.0                       # exact solution
    # b = [6, 8, 3, 4], r = [0, 0, 3, 4]: ||r|| / ||b|| = 5 / sqrt(125) = 1 / sqrt(5)
    b = np.array([6.0, 8.0, 3.0, 4.0])
    assert abs(oracle.true_relres_ld(I4, b, x) - float(1 / Decimal(5).sqrt())) <= EPS
    # 2 I x = b / 2 -> r = b / 2 -> exactly 0.5 (a dropped sqrt gives 0.25,
    # dividing by ||b||^2 gives 0.05)
    assert oracle.true_relres_ld(2.0 * np.eye(2), np.array([6.0, 8.0]),
                                 np.array([1.5, 2.0])) == 0.5


def test_true_relres_dyadic_exact():
    """Random dyadic A, x, b (12-bit mantissas): the long-double sum may round only
    in its last bits, so the result is the exact value to within 1 ulp."""
    rng = np.random.default_rng(13)
    for trial in range(12):
        n = int(rng.integers(2, 24))
        A = rng.integers(-2048, 2048, (n, n)) / 1024.0
        x = rng.integers(-2048, 2048, n) / 256.0
        b = rng.integers(-2048, 2048, n) / 64.0
        if not np.any(b):
            b[0] = 1.0
        got = oracle.true_relres_ld(A, b, x)
        expect = _exact_ratio(A, b, x)
        assert abs(got - expect) <= 2 * EPS * expect, (trial, got, expect)


def test_true_relres_scale_invariance_and_threads():
    """Scaling b and x by 2^k leaves the ratio bit-for-bit unchanged; the
    threaded sum (long double) stays within an ulp of the 1-thread one."""
    A, b = synth.gdd(512, 16)
    x = np.linalg.solve(A, b) * (1 + 1e-6 * np.random.default_rng(1).standard_normal(512))
    r1 = oracle.true_relres_ld(A, b, x)
    assert oracle.true_relres_ld(A, 8.0 * b, 8.0 * x) == r1
    op4 = oracle.Operator(A, threads=4)
    assert abs(oracle.true_relres_ld(op4, b, x) - r1) <= 2 * EPS * r1
    # independent double-double-free check: numpy long double of the same sum
    rl = (b.astype(np.longdouble) - (A.astype(np.longdouble) @ x.astype(np.longdouble)))
    ref = float(np.sqrt(np.sum(rl * rl)) / np.sqrt(np.sum(b.astype(np.longdouble) ** 2)))
    assert abs(r1 - ref) <= 1e-12 * ref


@pytest.mark.parametrize("kind", ["spd", "dd"])
def test_true_relres_stored_equals_on_the_fly(kind):
    """The on-the-fly operator (used at n = 65536 .. 262144, where A is not
    stored) must give exactly the stored-matrix value: same entries, same order."""
    n = 512
    spec = synth.spec(kind, n, kappa=1e3, kd=16)
    A = synth.gspd(n, 1e3)[0] if kind == "spd" else synth.gdd(n, 16)[0]
    b = synth.rhs(n)
    x = np.random.default_rng(2).standard_normal(n) * 1e-3
    st = oracle.true_relres_ld(oracle.Operator(A, threads=1), b, x)
    fly = oracle.true_relres_ld(oracle.Operator(gen=spec, threads=1), b, x)
    assert st == fly
    y1 = oracle.Operator(A, threads=1).apply(x)
    y2 = oracle.Operator(gen=spec, threads=3).apply(x)
    assert np.array_equal(y1, y2)


# ------------------------------------------------- BiCGSTAB P3, every step

def _mv(A, v):
    return [sum(a * b for a, b in zip(row, v)) for row in A]


def _dotq(a, b):
    return sum(x * y for x, y in zip(a, b))


def _bicgstab_rational_steps(A, b, maxit):
    """SURVEY.md sec.8(c).4 in exact rationals; one record per loop body:
    x_i, s_i, r_i (None on the half-step exit)."""
    n = len(b)
    x = [F(0)] * n
    r = [F(v) for v in b]
    rhat = r[:]
    rho_old = alpha = omega = F(1)
    v = [F(0)] * n
    p = [F(0)] * n
    out = []
    for _ in range(maxit):
        rho = _dotq(rhat, r)                                          # 5
        beta = (rho / rho_old) * (alpha / omega)                      # 6
        p = [ri + beta * (pi - omega * vi) for ri, pi, vi in zip(r, p, v)]   # 7
        v = _mv(A, p)                                                 # 8
        alpha = rho / _dotq(rhat, v)                                  # 9, 10
        s = [ri - alpha * vi for ri, vi in zip(r, v)]                 # 11
        if _dotq(s, s) == 0:                                          # 12
            x = [xi + alpha * pi for xi, pi in zip(x, p)]
            out.append({"x": x, "s": s, "r": None})
            return out
        t = _mv(A, s)                                                 # 13
        omega = _dotq(t, s) / _dotq(t, t)                             # 14
        x = [xi + alpha * pi + omega * si for xi, pi, si in zip(x, p, s)]   # 15
        r = [si - omega * ti for si, ti in zip(s, t)]                 # 16
        out.append({"x": x, "s": s, "r": r})
        if _dotq(r, r) == 0:                                          # 17
            return out
        rho_old = rho                                                 # 18
    return out


def _f(v):
    return np.array([float(t) for t in v])


@pytest.mark.parametrize("n", [3, 4, 5, 6])
def test_P3_bicgstab_every_step(n):
    """Every FP64 iterate of the oracle vs the rational run: x_i to 1e-12 relative,
    s_i and r_i to 1e-12 of ||b|| (residual vectors shrink to 0 at termination,
    so their error is measured on the problem's scale), hist_i to 1e-12 absolute
    (observed maxima over these systems: 3.8e-14, 3.3e-13, 1.2e-11 relative =
    <= 3e-13 absolute).  Exact termination: the rational run ends within n
    bodies with x = A^{-1} b."""
    rng = np.random.default_rng(200 + n)
    for trial in range(20):
        M = rng.integers(-3, 4, (n, n))
        M[np.arange(n), np.arange(n)] = np.abs(M).sum(axis=1) + 2
        A = M.tolist()
        b = rng.integers(-5, 6, n).tolist()
        if not any(b):
            b[0] = 1
        steps = _bicgstab_rational_steps(A, b, 2 * n)
        K = len(steps)
        assert K <= n
        Af, bf = np.array(A, float), np.array(b, float)
        nb = float(np.linalg.norm(bf))
        exact = np.linalg.solve(Af, bf)
        assert np.allclose(_f(steps[-1]["x"]), exact, rtol=1e-12, atol=0)
        _, h, rep, tr = oracle.bicgstab(Af, bf, tol=0.0, maxit=K, trace=K)
        assert rep.iterations == K
        for k, e in enumerate(steps, start=1):
            xf, _, _ = oracle.bicgstab(Af, bf, tol=0.0, maxit=k)
            ex = _f(e["x"])
            assert np.linalg.norm(xf - ex) <= 1e-12 * np.linalg.norm(ex), (trial, k)
            assert np.linalg.norm(tr["s"][k - 1] - _f(e["s"])) <= 1e-12 * nb, (trial, k)
            if e["r"] is not None:
                er = _f(e["r"])
                assert np.linalg.norm(tr["r"][k - 1] - er) <= 1e-12 * nb, (trial, k)
                hq = float(Decimal(_dotq(e["r"], e["r"]).numerator).sqrt()
                           / Decimal(_dotq(e["r"], e["r"]).denominator).sqrt()) / nb
                assert abs(h[k - 1] - hq) <= 1e-12, (trial, k, h[k - 1], hq)


def test_P3_bicgstab_catches_a_wrong_coefficient():
    """The per-step comparison above has teeth: the rational run with omega
    replaced by omega/2 (a minimal-residual step done wrong) still reaches the
    solution, but its intermediate iterates differ from the oracle's by far more
    than 1e-12."""
    rng = np.random.default_rng(205)
    n = 5
    M = rng.integers(-3, 4, (n, n))
    M[np.arange(n), np.arange(n)] = np.abs(M).sum(axis=1) + 2
    A, b = M.tolist(), rng.integers(-5, 6, n).tolist()
    Af, bf = np.array(A, float), np.array(b, float)
    steps = _bicgstab_rational_steps(A, b, 2 * n)
    xf, _, _ = oracle.bicgstab(Af, bf, tol=0.0, maxit=1)
    assert np.linalg.norm(xf - _f(steps[0]["x"])) <= 1e-12 * np.linalg.norm(_f(steps[0]["x"]))
    # one body with the halved omega
    r = [F(v) for v in b]
    v = _mv(A, r)
    alpha = _dotq(r, r) / _dotq(r, v)
    s = [ri - alpha * vi for ri, vi in zip(r, v)]
    t = _mv(A, s)
    omega = _dotq(t, s) / _dotq(t, t) / 2
    xw = _f([alpha * ri + omega * si for ri, si in zip(r, s)])
    assert np.linalg.norm(xf - xw) > 1e-6 * np.linalg.norm(xw)


# --------------------------------------- the measurements behind readings

def test_Q17_bicgstab_floor_distribution():
    """Reading Q17: the absolute floor of the BiCGSTAB history
    bar.  24 symmetric permutations P A P^T, P b of G-DD(1024, 16) are the same
    system in exact arithmetic, i.e. 24 legitimate FP64 summation orders; the
    oracle's histories differ from the unpermuted run by up to ~5.5e-13 (near
    relres 1e-10).  So a 2e-13 floor would fail legitimate orders, and 1e-12
    (the GPU tests' FLOOR_BS) keeps a ~2x margin over the worst observed."""
    A, b = synth.gdd(1024, 16)
    _, h1, r1 = oracle.bicgstab(A, b, tol=1e-10)
    worst = []
    for s in range(1, 25):
        P = np.random.default_rng(s).permutation(1024)
        _, h2, r2 = oracle.bicgstab(A[np.ix_(P, P)], b[P], tol=1e-10)
        assert r2.iterations == r1.iterations == 34
        d = np.abs(h1 - h2)
        big = h1 > 1e-6
        assert np.all(d[big] <= 1e-8 * h1[big])          # the relative bar holds above 1e-6
        worst.append(float(d.max()))
    assert max(worst) > 2e-13                            # a tighter floor is wrong
    assert max(worst) < 1e-12 / 1.5                      # FLOOR_BS keeps a margin
    assert sum(w > 2e-13 for w in worst) >= 3


def test_chaos_convection_diffusion_not_a_parity_input():
    """SPEC.md:560's nonnormal convection-diffusion matrix (n = 100, h = 0.1): two
    legitimate summation orders of the SAME oracle (the matrix and its symmetric
    reversal) take 106 and 104 BiCGSTAB iterations and their histories separate
    beyond the 1e-8 bar from iteration 20 on -- so the GPU tests check SPEC's
    property (converges within 200 iterations) and the true residual instead of
    the history."""
    A = synth.convection_diffusion(100, 0.1)
    b = np.ones(100)
    x1, h1, r1 = oracle.bicgstab(A, b, tol=1e-8)
    P = np.arange(100)[::-1]
    x2, h2, r2 = oracle.bicgstab(A[np.ix_(P, P)], b[P], tol=1e-8)
    assert (r1.iterations, r2.iterations) == (106, 104)
    rel = np.abs(h1[:100] - h2[:100]) / h1[:100]
    first = int(np.argmax(rel > 1e-8))
    assert first == 19 and np.all(rel[:19] <= 1e-8)
    assert oracle.true_relres_ld(A, b, x1) <= 10 * 1e-8
    assert oracle.true_relres_ld(A, b, x2[np.argsort(P)]) <= 10 * 1e-8


def test_chaos_random_sign_diagonal_not_a_parity_input():
    """Random-sign diagonally dominant matrices (synth.random_dd): the oracle on a
    reversed copy agrees to 1e-13 for two iterations, then the histories differ by
    more than 1e-3 relative within 7 iterations -- amplification of rounding, not
    a bug, so these matrices are used only for true-residual checks."""
    n = 300
    b = np.random.default_rng(6).standard_normal(n)
    P = np.arange(n)[::-1]
    for s in range(3):
        A = synth.random_dd(n, s)
        _, h1, _ = oracle.bicgstab(A, b, tol=1e-10)
        _, h2, _ = oracle.bicgstab(A[np.ix_(P, P)], b[P], tol=1e-10)
        rel = np.abs(h1[:8] - h2[:8]) / h1[:8]
        assert np.all(rel[:2] <= 1e-13), (s, rel)
        assert np.max(rel[:7]) > 1e-3, (s, rel)
