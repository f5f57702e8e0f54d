"""Pins for the oracle's BiCG and GMRES(m) -- the paper's other Krylov methods
(listed as implemented at PAPER.md:78, 109)."""
import json
import os
from fractions import Fraction as F

import numpy as np
import pytest

import oracle
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold():
    with open(os.path.join(GOLD, "spec_examples.json")) as f:
        return json.load(f)


def _mv(A, v):
    return [sum(a * b for a, b in zip(row, v)) for row in A]


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


# ----------------------------------------------------------------- gemv_t
def test_gemv_t_exact_on_integers():
    rng = np.random.default_rng(11)
    for m, n in [(1, 1), (5, 3), (17, 33)]:
        A = rng.integers(-20, 20, (m, n)).astype(float)
        x = rng.integers(-20, 20, m).astype(float)
        exact = [sum(F(int(A[i, j])) * int(x[i]) for i in range(m)) for j in range(n)]
        assert [F(v) for v in oracle.gemv_t(A, x)] == exact


# ------------------------------------------------------------------- BiCG
def test_bicg_spec_examples():
    for e in _gold()["bicg"]:
        x, h, r = oracle.bicg(np.array(e["A"], float), e["b"], tol=1e-12)
        assert r.converged and r.iterations <= e["max_iterations"], e["cite"]
        assert np.allclose(x, e["x"], rtol=1e-12, atol=0), e["cite"]


def test_bicg_equals_cg_on_spd():
    """with rt0 = r0 on SPD A, BiCG's iterates are CG's (the shadow
    sequence equals the primal one).  CG's oracle is itself pinned."""
    for A, b in [(np.diag([1.0, 2.0, 3.0]), np.ones(3)), (synth.gspd(256, 100.0)[0], synth.rhs(256))]:
        for k in (1, 2, 5, 20):
            xb, hb, rb = oracle.bicg(A, b, tol=0.0, maxit=k)
            xc, hc, rc = oracle.cg(A, b, tol=0.0, maxit=k)
            if rc.iterations < k:
                continue
            assert np.linalg.norm(xb - xc) <= 1e-10 * np.linalg.norm(xc)


@pytest.mark.parametrize("n", [3, 4, 5])
def test_bicg_exact_termination(n):
    """Exact arithmetic: BiCG on a nonsymmetric system reaches the exact solution
    in <= n steps (two Krylov spaces of dimension n); the FP64 oracle agrees."""
    rng = np.random.default_rng(300 + n)
    for trial in range(3):
        M = rng.integers(-3, 4, (n, n))
        M[np.arange(n), np.arange(n)] = np.abs(M).sum(axis=1) + 2
        A = M.tolist()
        b = rng.integers(-5, 6, n).tolist() or [1]
        if not any(b):
            b[0] = 1
        # rational BiCG
        x = [F(0)] * n
        r = [F(v) for v in b]
        rt, p, pt = r[:], r[:], r[:]
        rho = sum(a * c for a, c in zip(rt, r))
        AT = [list(col) for col in zip(*A)]
        steps = 0
        for _ in range(n):
            q, qt = _mv(A, p), _mv(AT, pt)
            alpha = rho / sum(a * c for a, c in zip(pt, q))
            x = [a + alpha * c for a, c in zip(x, p)]
            r = [a - alpha * c for a, c in zip(r, q)]
            rt = [a - alpha * c for a, c in zip(rt, qt)]
            steps += 1
            if not any(r):
                break
            rho1 = sum(a * c for a, c in zip(rt, r))
            p = [a + rho1 / rho * c for a, c in zip(r, p)]
            pt = [a + rho1 / rho * c for a, c in zip(rt, pt)]
            rho = rho1
        assert not any(r) and steps <= n and x == _ge_exact(A, b)
        xf, _, rep = oracle.bicg(np.array(A, float), np.array(b, float), tol=1e-13)
        ex = np.array([float(v) for v in x])
        assert rep.converged and np.linalg.norm(xf - ex) <= 1e-12 * np.linalg.norm(ex)


def test_bicg_invariants_paper():
    """'two mutually orthogonal sequences of residual vectors and
    A-orthogonal sequences of direction vectors': <rt_i, r_j> = 0 and
    <pt_i, A p_j> = 0 for i != j (normalised, first 20 steps)."""
    A, b = synth.gdd(512, 4)
    K = 16
    x, h, rep, tr = oracle.bicg(A, b, tol=1e-10, trace=K)
    assert rep.iterations >= K
    R, RT, Pm, PT = tr["r"], tr["rt"], tr["p"], tr["pt"]
    G = RT @ R.T
    nrm = np.outer(np.linalg.norm(RT, axis=1), np.linalg.norm(R, axis=1))
    off = np.abs(G / nrm - np.diag(np.diag(G / nrm)))
    assert off.max() <= 1e-10
    C = PT @ (Pm @ A.T).T
    nrm = np.outer(np.linalg.norm(PT, axis=1), np.linalg.norm(Pm @ A.T, axis=1))
    off = np.abs(C / nrm - np.diag(np.diag(C / nrm)))
    assert off.max() <= 1e-10


def test_bicg_gdd_vs_ge_and_edges():
    A, b = synth.gdd(1024, 4)
    x, h, rep = oracle.bicg(A, b, tol=1e-10)
    xge = oracle.ge_solve_ld(A, b)
    assert rep.converged and np.linalg.norm(x - xge) <= 10 * 4.4 * 1e-10 * np.linalg.norm(xge)
    assert oracle.true_relres_ld(A, b, x) <= 10 * 1e-10
    x, h, rep = oracle.bicg(A, np.zeros(1024), tol=1e-10)
    assert rep.converged and rep.iterations == 0 and np.all(x == 0)
    x, h, rep = oracle.bicg(np.array([[0.0, 1.0], [1.0, 0.0]]), [1.0, 0.0], tol=1e-12)
    assert rep.status == oracle.EBREAKDOWN and rep.iterations == 0     # <pt, A p> = 0


# ------------------------------------------------------------------ GMRES
def test_gmres_spec_examples():
    for e in _gold()["gmres"]:
        x, h, r = oracle.gmres(np.array(e["A"], float), e["b"], tol=1e-12, restart=e["restart"])
        assert r.converged and r.iterations <= e["max_iterations"], e["cite"]
        assert np.allclose(x, e["x"], rtol=1e-12, atol=1e-15), e["cite"]


def test_gmres_restart_stress_monotone():
    """A = diag(1..10), m = 2 converges with monotone per-cycle
    residuals; full GMRES (m = n) converges in <= n inner steps."""
    A = np.diag(np.arange(1.0, 11.0))
    b = np.ones(10)
    x, h, r = oracle.gmres(A, b, tol=1e-10, restart=2, maxit=1000)
    assert r.converged
    cycles = [h[i:i + 2] for i in range(0, len(h), 2)]
    assert all(np.all(np.diff(c) <= 0) for c in cycles)
    x, h, r = oracle.gmres(A, b, tol=1e-12, restart=10)
    assert r.converged and r.iterations <= 10
    assert np.all(np.diff(h) <= 0)


def test_gmres_minimal_residual_property():
    """GMRES's defining property: after k steps the residual is the minimum of
    ||b - A z|| over z in K_k(A, b) -- a least-squares problem solved here by
    LAPACK on an orthonormal Krylov basis (independent of the oracle)."""
    A, b = synth.gdd(200, 4)      # cond ~4.4: the power basis below stays well conditioned
    x, h, r = oracle.gmres(A, b, tol=0.0, restart=50, maxit=10)
    K = np.empty((200, 10))
    v = b / np.linalg.norm(b)
    for k in range(10):
        K[:, k] = v
        v = A @ v
        v /= np.linalg.norm(v)
    Q, _ = np.linalg.qr(K)
    for k in range(1, 11):
        AQ = A @ Q[:, :k]
        y, *_ = np.linalg.lstsq(AQ, b, rcond=None)
        best = np.linalg.norm(b - AQ @ y) / np.linalg.norm(b)
        assert abs(h[k - 1] - best) <= 1e-8 * best + 1e-14


def test_gmres_gdd_vs_ge_and_true_residual():
    A, b = synth.gdd(1024, 16)
    x, h, rep = oracle.gmres(A, b, tol=1e-10, restart=30)
    xge = oracle.ge_solve_ld(A, b)
    assert rep.converged
    assert np.linalg.norm(x - xge) <= 10 * 17.3 * 1e-10 * np.linalg.norm(xge)
    assert oracle.true_relres_ld(A, b, x) <= 10 * 1e-10
    x, h, rep = oracle.gmres(A, np.zeros(1024), tol=1e-10)
    assert rep.converged and rep.iterations == 0 and np.all(x == 0)
    x, h, rep = oracle.gmres(A, b, tol=1e-30, restart=5, maxit=12)
    assert rep.status == oracle.EMAXIT and rep.iterations == 12 and len(h) == 12
