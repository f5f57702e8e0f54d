"""Pins for the oracle's CG and BiCGSTAB (CPU only).

Each test pins the oracle to something other than itself: exact rationals,
the closed form, long-double Gaussian elimination (itself pinned to LAPACK),
finite termination, the invariants PAPER.md:33 states for the
BiCG family (residual orthogonality, A-conjugate directions), textbook bounds.
Pin numbers P1..P14 follow SURVEY.md sec.8(c).7.
"""
import json
import math
import os
from fractions import Fraction as F

import numpy as np
import pytest

import oracle
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")
EPS = 2.0 ** -52


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ------------------------------------------------------------ exact rationals

def _mv(A, v):
    return [sum(a * b for a, b in zip(row, v)) for row in A]


def _dotq(a, b):
    return sum(x * y for x, y in zip(a, b))


def _ge_exact(A, b):
    n = len(A)
    M = [list(map(F, row)) + [F(bi)] for row, bi in zip(A, b)]
    for k in range(n):
        piv = next(i for i in range(k, n) if M[i][k] != 0)
        M[k], M[piv] = M[piv], M[k]
        for i in range(k + 1, n):
            l = M[i][k] / M[k][k]
            M[i] = [a - l * c for a, c in zip(M[i], M[k])]
    x = [F(0)] * n
    for i in reversed(range(n)):
        x[i] = (M[i][n] - sum(M[i][j] * x[j] for j in range(i + 1, n))) / M[i][i]
    return x


def _cg_exact(A, b, steps):
    """Hestenes-Stiefel in exact rationals; returns iterates x_1..x_steps."""
    x = [F(0)] * len(b)
    r = [F(v) for v in b]
    p = r[:]
    rho = _dotq(r, r)
    xs = []
    for _ in range(steps):
        if rho == 0:
            break
        q = _mv(A, p)
        a = rho / _dotq(p, q)
        x = [xi + a * pi for xi, pi in zip(x, p)]
        r = [ri - a * qi for ri, qi in zip(r, q)]
        rho1 = _dotq(r, r)
        xs.append((x, rho1))
        p = [ri + (rho1 / rho) * pi for ri, pi in zip(r, p)]
        rho = rho1
    return xs


def test_P1_cg_textbook_2x2():
    g = _gold("cg_2x2_textbook.json")
    A = np.array(g["A"], float)
    x1, _, r1 = oracle.cg(A, g["b"], x0=g["x0"], tol=0.0, maxit=1)
    x2, hist, r2 = oracle.cg(A, g["b"], x0=g["x0"], tol=1e-14, maxit=10)
    for got, (p, q) in zip(x1, g["x1"]):
        assert abs(got - p / q) <= 4 * EPS * abs(p / q)
    for got, (p, q) in zip(x2, g["x2"]):
        assert abs(got - p / q) <= 4 * EPS * abs(p / q)
    assert r1.iterations == 1 and r1.status == oracle.EMAXIT
    assert r2.converged and r2.iterations == 2


def test_P2_spec_cg_examples():
    for e in _gold("spec_examples.json")["cg"]:
        A = np.array(e["A"], float)
        x, hist, rep = oracle.cg(A, e["b"], tol=1e-12)
        assert rep.converged, e["cite"]
        assert rep.iterations <= e["max_iterations"], e["cite"]
        assert np.allclose(x, e["x"], rtol=1e-12, atol=0), e["cite"]


def test_P2_spec_bicgstab_examples():
    for e in _gold("spec_examples.json")["bicgstab"]:
        if "cd_n" in e:
            A = synth.convection_diffusion(e["cd_n"], e["cd_h"])
            b = np.ones(e["cd_n"])
            x, hist, rep = oracle.bicgstab(A, b, tol=e["tol"])
            assert rep.converged and rep.iterations <= e["max_iterations"], e["cite"]
            xd = oracle.ge_solve_ld(A, b)
            assert np.linalg.norm(x - xd) / np.linalg.norm(xd) < 1e-6
            continue
        A = np.array(e["A"], float)
        x, hist, rep = oracle.bicgstab(A, e["b"], tol=1e-12)
        assert rep.converged and rep.iterations <= e["max_iterations"], e["cite"]
        assert np.allclose(x, e["x"], rtol=1e-12, atol=0), e["cite"]
    # [[2,1],[0,3]] b=[3,3] exits at the half step of iteration 1 (App. A.6)
    x, hist, rep = oracle.bicgstab(np.array([[2.0, 1.0], [0.0, 3.0]]), [3.0, 3.0], tol=1e-12)
    assert rep.half_step_exit and rep.iterations == 1 and rep.matvecs == 1


@pytest.mark.parametrize("n", [3, 4, 5, 6])
def test_P3_cg_exact_termination_and_fp64_agreement(n):
    """CG 'in exact arithmetic gives the solution for at most n
    iterations'.  The rational run must hit r = 0 by step n with x = A^{-1} b
    (exact GE); the FP64 oracle must follow the rational iterates to 1e-12."""
    rng = np.random.default_rng(100 + n)
    for trial in range(3):
        M = rng.integers(-3, 4, (n, n))
        A = (M.T @ M + np.eye(n, dtype=int)).tolist()
        b = rng.integers(-5, 6, n).tolist()
        if not any(b):
            b[0] = 1
        xs = _cg_exact(A, b, n)
        assert xs[-1][1] == 0 and len(xs) <= n
        assert xs[-1][0] == _ge_exact(A, b)
        Af = np.array(A, float)
        for k, (xk, _) in enumerate(xs, start=1):
            xf, _, _ = oracle.cg(Af, np.array(b, float), tol=0.0, maxit=k)
            ex = np.array([float(v) for v in xk])
            assert np.linalg.norm(xf - ex) <= 1e-12 * np.linalg.norm(ex)


def _bicgstab_exact(A, b, maxit):
    n = len(b)
    x = [F(0)] * n
    r = [F(v) for v in b]
    rhat = r[:]
    rho_old = alpha = omega = F(1)
    v = [F(0)] * n
    p = [F(0)] * n
    for i in range(1, maxit + 1):
        rho = _dotq(rhat, r)
        beta = (rho / rho_old) * (alpha / omega)
        p = [ri + beta * (pi - omega * vi) for ri, pi, vi in zip(r, p, v)]
        v = _mv(A, p)
        alpha = rho / _dotq(rhat, v)
        s = [ri - alpha * vi for ri, vi in zip(r, v)]
        if _dotq(s, s) == 0:
            x = [xi + alpha * pi for xi, pi in zip(x, p)]
            return x, i, True
        t = _mv(A, s)
        omega = _dotq(t, s) / _dotq(t, t)
        x = [xi + alpha * pi + omega * si for xi, pi, si in zip(x, p, s)]
        r = [si - omega * ti for si, ti in zip(s, t)]
        if _dotq(r, r) == 0:
            return x, i, False
        rho_old = rho
    return x, maxit, False


@pytest.mark.parametrize("n", [3, 4, 5])
def test_P3_bicgstab_exact_termination(n):
    """Exact arithmetic: BiCGSTAB reaches the exact solution within n iterations
    (Krylov dimension); the FP64 oracle matches it to 1e-12."""
    rng = np.random.default_rng(200 + n)
    for trial in range(3):
        M = rng.integers(-3, 4, (n, n))
        M[np.arange(n), np.arange(n)] = np.abs(M).sum(axis=1) + 2
        A = M.tolist()
        b = rng.integers(-5, 6, n).tolist()
        if not any(b):
            b[0] = 1
        x, iters, half = _bicgstab_exact(A, b, 2 * n)
        assert x == _ge_exact(A, b) and iters <= n
        xf, _, rep = oracle.bicgstab(np.array(A, float), np.array(b, float), tol=1e-13)
        ex = np.array([float(v) for v in x])
        assert rep.converged
        assert np.linalg.norm(xf - ex) <= 1e-12 * np.linalg.norm(ex)


def test_P4_finite_termination_fp64_diagonal():
    """diagonal SPD n <= 50 converges to 1e-12 in <= n iterations."""
    for seed in range(20):
        rng = np.random.default_rng(seed)
        n = int(rng.integers(2, 51))
        A = np.diag(rng.uniform(1.0, 10.0, n))
        b = rng.uniform(-1.0, 1.0, n)
        x, hist, rep = oracle.cg(A, b, tol=1e-12)
        assert rep.converged and rep.iterations <= n


# ------------------------------------------------- brute force / closed form

def test_ge_ld_pinned_to_lapack_and_residual():
    rng = np.random.default_rng(5)
    for n in (1, 2, 17, 200):
        A = rng.standard_normal((n, n)) + n * np.eye(n)
        b = rng.standard_normal(n)
        x = oracle.ge_solve_ld(A, b)
        xl = np.linalg.solve(A, b)
        assert np.linalg.norm(x - xl) <= 1e-12 * np.linalg.norm(xl)
        assert oracle.true_relres_ld(A, b, x) < 1e-15
    # pivoting: zero leading entry
    x = oracle.ge_solve_ld(np.array([[0.0, 1.0], [1.0, 0.0]]), [2.0, 3.0])
    assert x.tolist() == [3.0, 2.0]


def test_P5_P6_cg_c1_vs_ge_and_closed_form():
    """C1: G-SPD(1024, 1e3), tol 1e-10.  x vs long-double GE and the closed form,
    bound kappa*tol (P5/P6); GE vs closed form pins the generator too."""
    A, c, b = synth.gspd(1024, 1e3)
    x, hist, rep = oracle.cg(A, b, tol=1e-10)
    xge = oracle.ge_solve_ld(A, b)
    xcf = oracle.spd_exact_solve_ld(c, synth.SEED, b)
    assert np.linalg.norm(xge - xcf) <= 1e-14 * np.linalg.norm(xcf)
    assert np.linalg.norm(x - xcf) <= 1e3 * 1e-10 * np.linalg.norm(xcf)
    assert rep.converged
    assert oracle.true_relres_ld(A, b, x) <= 10 * 1e-10      # P11


def test_closed_form_residual_on_larger_n():
    n = 4096
    c = synth.spd_table(n, 1e4)
    b = synth.rhs(n)
    op = oracle.Operator(gen=synth.spec("spd", n, kappa=1e4), threads=4)
    x = oracle.spd_exact_solve_ld(c, synth.SEED, b)
    assert oracle.true_relres_ld(op, b, x) < 1e-12


def test_P5_bicgstab_gdd_vs_ge():
    for kd in (4, 16):
        A, b = synth.gdd(1024, kd)
        x, hist, rep = oracle.bicgstab(A, b, tol=1e-10)
        xge = oracle.ge_solve_ld(A, b)
        assert rep.converged
        assert np.linalg.norm(x - xge) <= 10 * 1.03 * kd * 1e-10 * np.linalg.norm(xge)
        assert oracle.true_relres_ld(A, b, x) <= 10 * 1e-10


# ---------------------------------------------------------------- invariants

def test_P7_cg_invariants():
    """PAPER.md:33 (BiCG family: mutually orthogonal residuals, A-orthogonal
    directions, 'similar to those of the CG method'); monotone A-norm error
    (Golub & Van Loan, ref [9]).  First 50 iterations, 1e-12."""
    A, c, b = synth.gspd(1024, 1e3)
    K = 51
    x, hist, rep, tr = oracle.cg(A, b, tol=1e-10, trace=K)
    R, P, X = tr["r"], tr["p"], tr["x"]
    Rn = R / np.linalg.norm(R, axis=1)[:, None]
    G = Rn @ Rn.T
    off = G - np.diag(np.diag(G))
    assert np.max(np.abs(off)) <= 1e-12
    AP = P @ A
    PAP = P @ AP.T
    d = np.sqrt(np.diag(PAP))
    C = PAP / np.outer(d, d)
    assert np.max(np.abs(C - np.diag(np.diag(C)))) <= 1e-12
    xs = oracle.spd_exact_solve_ld(c, synth.SEED, b)
    E = X - xs
    anorm = np.einsum("ij,ij->i", E, E @ A)
    assert np.all(np.diff(anorm) < 0)


def test_P8_bicgstab_invariants():
    """omega is a 1-D minimal-residual step: ||r_i|| <= ||s_i||; with rhat = r0
    on SPD A the first half step equals CG's first residual."""
    A, b = synth.gdd(1024, 16)
    x, hist, rep, tr = oracle.bicgstab(A, b, tol=1e-10, trace=40)
    k = rep.iterations - (1 if rep.half_step_exit else 0)
    for i in range(k):
        assert np.linalg.norm(tr["r"][i]) <= np.linalg.norm(tr["s"][i]) * (1 + 1e-14)
    As, c, bs = synth.gspd(256, 100.0)
    _, _, _, trc = oracle.cg(As, bs, tol=0.0, maxit=1, trace=2)
    _, _, _, trb = oracle.bicgstab(As, bs, tol=0.0, maxit=1, trace=1)
    assert np.linalg.norm(trb["s"][0] - trc["r"][1]) <= 1e-14 * np.linalg.norm(trc["r"][1])


def test_P10_cg_iteration_bound():
    for n, kappa in [(1024, 1e3), (1024, 1e4)]:
        A, c, b = synth.gspd(n, kappa)
        _, _, rep = oracle.cg(A, b, tol=1e-10)
        sk = math.sqrt(kappa)
        bound = math.ceil(math.log(2 * sk / 1e-10) / math.log((sk + 1) / (sk - 1)))
        assert rep.iterations <= bound


# ---------------------------------------------------- survey App. A.8 (P14)

def test_P14_survey_spec_numbers():
    g = _gold("survey_a8.json")
    for e in g["cg"]:
        A, c, b = synth.gspd(e["n"], e["kappa"])
        x, hist, rep = oracle.cg(A, b, tol=1e-10)
        assert rep.iterations == e["iterations"]
        assert np.allclose(hist[:3], e["hist0"], rtol=5e-7, atol=0)
    for e in g["bicgstab"]:
        A, b = synth.gdd(e["n"], e["kd"])
        x, hist, rep = oracle.bicgstab(A, b, tol=1e-10)
        assert rep.iterations == e["iterations"]
        assert rep.half_step_exit == e["half_step_exit"]


# ------------------------------------------------------------- edge cases

def test_edge_b_zero_and_exact_start():
    A = synth.random_spd(8, 10.0, 0)
    for fn in (oracle.cg, oracle.bicgstab):
        x, hist, rep = fn(A, np.zeros(8), x0=np.ones(8), tol=1e-10)
        assert rep.converged and rep.iterations == 0 and np.all(x == 0)
    xs = np.linalg.solve(A, np.ones(8))
    b = A @ xs
    x, hist, rep = oracle.cg(A, b, x0=xs, tol=1e-6)
    assert rep.iterations == 0 and np.array_equal(x, xs)


def test_edge_notspd_and_breakdown_and_maxit():
    A = np.diag([1.0, -1.0])
    x, hist, rep = oracle.cg(A, [1.0, 1.0], tol=1e-12)
    assert rep.status == oracle.ENOTSPD and rep.iterations == 0
    R = np.array([[0.0, 1.0], [-1.0, 0.0]])      # <rhat, A r0> = 0 at iteration 1
    x, hist, rep = oracle.bicgstab(R, [1.0, 0.0], tol=1e-12)
    assert rep.status == oracle.EBREAKDOWN and rep.iterations == 0 and np.all(x == 0)
    A, c, b = synth.gspd(1024, 1e3)
    x, hist, rep = oracle.cg(A, b, tol=1e-10, maxit=7)
    assert rep.status == oracle.EMAXIT and rep.iterations == 7 and hist.size == 7
    x, hist, rep = oracle.cg(A, b, tol=1e-10, maxit=0)
    assert rep.status == oracle.EMAXIT and rep.iterations == 0 and np.all(x == 0)


def test_Q17_bicgstab_floor():
    """Reading Q17: the history bar needs an absolute floor because
    two legitimate FP64 evaluation orders of the SAME method differ at the
    rounding floor.  A symmetric permutation P A P^T, P b is the same system in
    exact arithmetic; the oracle's own histories on the two copies differ by
    > 1e-14 (so survey's 1e-14 floor is too tight for BiCGSTAB) but < 1e-12
    (the floor the GPU tests use), while the relative bar holds above 1e-6."""
    A, b = synth.gdd(1024, 16)
    _, h1, r1 = oracle.bicgstab(A, b, tol=1e-10)
    P = np.arange(1024)[::-1]
    _, h2, r2 = oracle.bicgstab(A[np.ix_(P, P)], b[P], tol=1e-10)
    assert r1.iterations == r2.iterations
    d = np.abs(h1 - h2)
    assert d.max() > 1e-14 and d.max() < 1e-12
    big = h1 > 1e-6
    assert np.all(d[big] <= 1e-8 * h1[big])
