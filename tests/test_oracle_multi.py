"""Pins for the oracle's multi-RHS CG (oracle.cg_multi, reading Q30): the
per-column recurrences against closed forms, with several right-hand sides in ONE
call so a column/layout mix-up (wrong column, transposed block, shared scalars)
fails.  CPU only."""
import numpy as np

import oracle

EPS = 2.0 ** -52


def test_diag_block_closed_forms():
    """SPEC.md:532 (diag(1,2,3), b = 1 -> [1, 1/2, 1/3]) next to b = A [2,2,2] and
    b = 0 (Q6: x = 0, 0 iterations) in one block."""
    A = np.diag([1.0, 2.0, 3.0])
    B = np.column_stack([np.ones(3), A @ np.full(3, 2.0), np.zeros(3)])
    X, hs, reps = oracle.cg_multi(A, B, tol=1e-14)
    assert np.allclose(X[:, 0], [1.0, 0.5, 1.0 / 3.0], rtol=4 * EPS, atol=0)
    assert np.allclose(X[:, 1], [2.0, 2.0, 2.0], rtol=4 * EPS, atol=0)
    assert np.all(X[:, 2] == 0) and reps[2].iterations == 0 and reps[2].converged
    assert reps[0].iterations <= 3 and reps[1].iterations <= 3
    assert len(hs[0]) == reps[0].iterations


def test_textbook_2x2_and_second_column():
    """P1's 2 x 2 system (x* = [1/11, 7/11]) and b = A [1, 1] = [5, 4] (x* = [1, 1])
    in one block: both reach their own exact solution in 2 steps."""
    A = np.array([[4.0, 1.0], [1.0, 3.0]])
    B = np.array([[1.0, 5.0], [2.0, 4.0]])
    X, hs, reps = oracle.cg_multi(A, B, tol=1e-15)
    assert np.allclose(X[:, 0], [1 / 11, 7 / 11], rtol=8 * EPS, atol=0)
    assert np.allclose(X[:, 1], [1.0, 1.0], rtol=8 * EPS, atol=0)
    assert all(r.iterations <= 2 for r in reps)


def test_column_permutation_is_a_permutation():
    """Column independence: permuting B permutes X, the histories and the reports
    bitwise (no cross-column scalar)."""
    rng = np.random.default_rng(7)
    n = 40
    M = rng.standard_normal((n, n))
    A = M @ M.T + n * np.eye(n)
    B = rng.standard_normal((n, 5))
    X, hs, reps = oracle.cg_multi(A, B, tol=1e-12)
    perm = [3, 0, 4, 1, 2]
    Xp, hsp, repsp = oracle.cg_multi(A, B[:, perm], tol=1e-12)
    assert np.array_equal(Xp, X[:, perm])
    for j, k in enumerate(perm):
        assert np.array_equal(hsp[j], hs[k]) and repsp[j].iterations == reps[k].iterations


def test_per_column_notspd_and_x0():
    """A = diag(1, -1): b = e1 lives in the positive eigenspace (1 step, exact),
    b = e2 meets <p, A p> = -1 < 0 at k = 1 (NOTSPD, x = x0 unchanged) -- per column."""
    A = np.diag([1.0, -1.0])
    B = np.array([[1.0, 0.0], [0.0, 1.0]])
    X0 = np.zeros((2, 2))
    X, hs, reps = oracle.cg_multi(A, B, X0=X0, tol=1e-12)
    assert reps[0].status == oracle.OK and reps[0].iterations == 1 and np.array_equal(X[:, 0], [1.0, 0.0])
    assert reps[1].status == oracle.ENOTSPD and reps[1].iterations == 0 and np.all(X[:, 1] == 0)


def test_bicgstab_multi_spec_example_and_second_column():
    """SPEC.md:559 ([[2,1],[0,3]] x = [3,3] -> [1,1], a half-step exit at iteration 1)
    next to b = A [1, 2] = [4, 6] and b = 0, in one block."""
    A = np.array([[2.0, 1.0], [0.0, 3.0]])
    B = np.array([[3.0, 4.0, 0.0], [3.0, 6.0, 0.0]])
    X, hs, reps = oracle.bicgstab_multi(A, B, tol=1e-14)
    assert np.allclose(X[:, 0], [1.0, 1.0], rtol=8 * EPS, atol=0)
    assert reps[0].iterations == 1 and reps[0].half_step_exit
    assert np.allclose(X[:, 1], [1.0, 2.0], rtol=8 * EPS, atol=0)
    assert np.all(X[:, 2] == 0) and reps[2].iterations == 0 and reps[2].converged


def test_bicgstab_multi_per_column_breakdown():
    """A = diag(2, 2) (+) [[0, 1], [-1, 0]]: b = e1 lies in the diagonal block (one
    half step, exact), b = e3 in the rotation block meets <rhat, A r0> = <e3, -e4> = 0
    at iteration 1 (BREAKDOWN, 0 iterations, x = 0) -- per column."""
    A = np.zeros((4, 4))
    A[0, 0] = A[1, 1] = 2.0
    A[2, 3], A[3, 2] = 1.0, -1.0
    B = np.zeros((4, 2))
    B[0, 0] = 1.0
    B[2, 1] = 1.0
    X, hs, reps = oracle.bicgstab_multi(A, B, tol=1e-14)
    assert reps[0].status == oracle.OK and np.allclose(X[:, 0], [0.5, 0, 0, 0], rtol=0, atol=4 * EPS)
    assert reps[1].status == oracle.EBREAKDOWN and reps[1].iterations == 0 and np.all(X[:, 1] == 0)


def test_bicgstab_multi_column_permutation():
    rng = np.random.default_rng(11)
    n = 30
    A = rng.standard_normal((n, n)) + n * np.eye(n)
    B = rng.standard_normal((n, 4))
    X, hs, reps = oracle.bicgstab_multi(A, B, tol=1e-12)
    perm = [2, 0, 3, 1]
    Xp, hsp, repsp = oracle.bicgstab_multi(A, B[:, perm], tol=1e-12)
    assert np.array_equal(Xp, X[:, perm])
    for j, k in enumerate(perm):
        assert np.array_equal(hsp[j], hs[k]) and repsp[j].iterations == reps[k].iterations
