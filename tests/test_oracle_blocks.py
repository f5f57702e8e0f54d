"""Pins for the oracle's building blocks and generators (CPU only).

Building blocks: SURVEY.md sec.8(c).1 ("inner products, saxpy and
matrix-vector products").  Generators: SURVEY.md sec.8(d).2, pin P12.
"""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def test_spec_axpy_dot_nrm2_gemv():
    g = _gold("spec_examples.json")
    for e in g["axpy"]:
        assert oracle.axpy(e["alpha"], e["x"], e["y"]).tolist() == e["out"], e["cite"]
    for e in g["dot"]:
        assert oracle.dot(e["x"], e["y"]) == e["out"], e["cite"]
    for e in g["nrm2"]:
        assert oracle.nrm2(e["x"]) == e["out"], e["cite"]
    for e in g["gemv"]:
        assert oracle.gemv(np.array(e["A"], float), e["x"]).tolist() == e["out"], e["cite"]


def test_gemv_exact_on_integers_vs_fractions():
    """Brute force: small-integer entries make every partial sum exact in FP64,
    so the oracle must equal the exact rational product (catches transposed
    operands, dropped terms, wrong strides)."""
    rng = np.random.default_rng(1)
    for m, n in [(1, 1), (3, 5), (7, 4), (33, 65)]:
        A = rng.integers(-50, 50, (m, n)).astype(float)
        x = rng.integers(-50, 50, n).astype(float)
        exact = [sum(Fraction(int(A[i, j])) * int(x[j]) for j in range(n)) for i in range(m)]
        y = oracle.gemv(A, x)
        assert [Fraction(v) for v in y] == exact


def test_gemv_row_major_nonsymmetric():
    A = np.array([[0.0, 1.0], [0.0, 0.0]])
    assert oracle.gemv(A, [0.0, 1.0]).tolist() == [1.0, 0.0]
    assert oracle.gemv(A, [1.0, 0.0]).tolist() == [0.0, 0.0]


def test_gemv_sequential_order_and_thread_invariance():
    """Rows are summed left to right without FMA: (1e16 + 1) - 1e16 = 0 in FP64
    sequential order, while a reordered sum would give 1 (fixes c.2 rule)."""
    A = np.array([[1e16, 1.0, -1e16], [1.0, 1e16, -1e16]])
    y = oracle.gemv(A, [1.0, 1.0, 1.0])
    assert y.tolist() == [0.0, 0.0]
    rng = np.random.default_rng(2)
    B = rng.standard_normal((301, 257))
    x = rng.standard_normal(257)
    y1 = oracle.gemv(B, x, threads=1)
    y4 = oracle.gemv(B, x, threads=4)
    assert np.array_equal(y1, y4)
    # sequential order exactly: compare with a Python left-to-right loop on a few rows
    for i in (0, 150, 300):
        s = 0.0
        for j in range(257):
            s += B[i, j] * x[j]
        assert y1[i] == s


def test_dot_matches_math_fsum_bound():
    import math
    rng = np.random.default_rng(3)
    x, y = rng.standard_normal(10000), rng.standard_normal(10000)
    exact = math.fsum((x * y).tolist())  # products rounded; sum exact
    d = oracle.dot(x, y)
    gamma = 10000 * 2.0 ** -53 / (1 - 10000 * 2.0 ** -53)
    assert abs(d - exact) <= 2 * gamma * float(np.abs(x * y).sum())


# ---------------------------------------------------------------- generators (P12)

def test_splitmix_reference_values():
    """SplitMix64 with seed 0 state stepping: the generator's published first
    output for state 0 is 0xE220A8397B1DCDAF (Vigna's splitmix64.c)."""
    assert int(synth.sm64(np.uint64(0))) == 0xE220A8397B1DCDAF
    for seed, stream, key in [(0, 0, 0), (151107174, 3, 17), (2 ** 63 + 5, 4, 2 ** 40 + 3)]:
        assert oracle.hash64(seed, stream, key) == int(synth.hash64(seed, stream, key))


@pytest.mark.parametrize("n,kappa", [(64, 10.0), (1024, 1e3), (2048, 1e4)])
def test_gspd_bitwise_and_properties(n, kappa):
    A, c, b = synth.gspd(n, kappa)
    sp = synth.spec("spd", n, kappa=kappa)
    assert np.array_equal(oracle.gen_rows(sp, 0, n), A)
    assert np.array_equal(oracle.gen_rhs(n, synth.SEED), b)
    assert np.array_equal(A, A.T)                      # exactly symmetric
    ev = np.linalg.eigvalsh(A)
    assert abs(ev[0] - 1.0) < 1e-9 * kappa and abs(ev[-1] / ev[0] / kappa - 1) < 1e-9
    assert np.all(np.abs(b) < 1.0)


@pytest.mark.parametrize("n,kd", [(5, 1), (257, 4), (1000, 16), (1024, 1024)])
def test_gdd_bitwise_and_dominance(n, kd):
    A, b = synth.gdd(n, kd)
    sd = synth.spec("dd", n, kd=kd)
    assert np.array_equal(oracle.gen_rows(sd, 0, n), A)
    assert np.array_equal(oracle.gen_rows(sd, n // 3, n // 2), A[n // 3: n // 3 + n // 2])
    off = np.abs(A).sum(axis=1) - np.abs(np.diag(A))
    # dominance margin >= 1/16 and row sums exact in reversed order
    assert np.all(np.abs(np.diag(A)) >= off * 17 / 16)
    R_fwd = [sum(abs(v) for j, v in enumerate(row) if j != i) for i, row in enumerate(A)]
    R_rev = [sum(abs(v) for j, v in reversed(list(enumerate(row))) if j != i)
             for i, row in enumerate(A)]
    assert R_fwd == R_rev


def test_rhs_is_exact_dyadic():
    b = synth.rhs(4096)
    assert np.all((b * 2.0 ** 53) == np.round(b * 2.0 ** 53))
    assert -1.0 <= b.min() and b.max() < 1.0
