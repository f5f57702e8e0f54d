"""Seeded synthetic inputs for the dense CG / BiCGSTAB path.

This module holds none of the method's arithmetic: it only builds A and b.  It is
the one module both sides may use -- the tests feed its host arrays to the CUDA
path (``ks_load_rows``) and to the oracle.  For the multi-GB configs the CUDA
library expands the same spec on the device (K0) and the oracle expands it on the
host with its own independent SplitMix64 (``oracle/ks_oracle.c``); pin P12 checks
that all three expansions are bitwise equal.

Generators (counter-based, O(1) per entry, exact):
  H(seed, stream, key) = sm64(sm64(seed ^ (stream << 56)) + key)        SplitMix64
  G-SPD(n, kappa, seed): A_ij = s_i s_j c[(i-j) mod n], c = (1/n) IDFT(lambda),
      lambda_0 = 1, lambda_{n/2} = kappa, lambda_k = lambda_{n-k} =
      1 + (kappa-1) U53(seed,3,k); s_i = 1 - 2 (H(seed,4,i) >> 63).
  G-DD(n, kd, seed): h_ij = ((H(seed,0,i*n+j) >> 44) - 2^19) 2^-20 (j != i),
      A_ii = R_i * 17/16 (1 + k_i), R_i = sum_{j != i} |h_ij|,
      k_i = (H(seed,1,i) >> 32) mod kd.
  b_i = 2 U53(seed,2,i) - 1;  x0 = 0.
Seeds: 151107174 (the arXiv id) and 1511071740.
"""
from __future__ import annotations

import numpy as np

SEED = 151107174
SEED2 = 1511071740

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def sm64(z):
    """SplitMix64 finaliser on a uint64 array (wraparound arithmetic)."""
    z = np.asarray(z, dtype=np.uint64).copy()
    with np.errstate(over="ignore"):
        z += np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def hash64(seed: int, stream: int, key) -> np.ndarray:
    base = sm64(np.uint64(seed) ^ (np.uint64(stream) << np.uint64(56)))
    with np.errstate(over="ignore"):
        return sm64(base + np.asarray(key, dtype=np.uint64))


def u53(seed: int, stream: int, key) -> np.ndarray:
    return (hash64(seed, stream, key) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def rhs(n: int, seed: int = SEED) -> np.ndarray:
    """b_i = 2 U53(seed, 2, i) - 1 (exact dyadic values in [-1, 1))."""
    return 2.0 * u53(seed, 2, np.arange(n, dtype=np.uint64)) - 1.0


def spd_eigenvalues(n: int, kappa: float, seed: int = SEED) -> np.ndarray:
    if n < 2 or n % 2:
        raise ValueError("G-SPD needs an even n >= 2")
    lam = np.empty(n)
    lam[0] = 1.0
    lam[n // 2] = kappa
    k = np.arange(1, n // 2, dtype=np.uint64)
    v = 1.0 + (kappa - 1.0) * u53(seed, 3, k)
    lam[1:n // 2] = v
    lam[n // 2 + 1:] = v[::-1]
    return lam


def spd_table(n: int, kappa: float, seed: int = SEED) -> np.ndarray:
    """Circulant first column c = (1/n) IDFT(lambda), symmetrised c[n-m] := c[m]."""
    lam = spd_eigenvalues(n, kappa, seed)
    c = np.fft.irfft(lam[: n // 2 + 1], n)
    c = np.ascontiguousarray(c, dtype=np.float64)
    m = np.arange(1, n // 2)
    c[n - m] = c[m]
    return c


def spd_signs(n: int, seed: int = SEED) -> np.ndarray:
    return np.where((hash64(seed, 4, np.arange(n, dtype=np.uint64)) >> np.uint64(63)) == 1,
                    -1.0, 1.0)


def gspd_rows(n: int, table: np.ndarray, seed: int, r0: int, r1: int) -> np.ndarray:
    """Rows [r0, r1) of G-SPD(n): A_ij = s_i s_j c[(i-j) mod n]."""
    s = spd_signs(n, seed)
    i = np.arange(r0, r1)[:, None]
    j = np.arange(n)[None, :]
    return (s[r0:r1, None] * s[None, :]) * table[(i - j) % n]


def gdd_rows(n: int, kd: int, seed: int, r0: int, r1: int) -> np.ndarray:
    """Rows [r0, r1) of G-DD(n, kd): exact dyadic off-diagonals, exact row sums."""
    i = np.arange(r0, r1, dtype=np.uint64)[:, None]
    j = np.arange(n, dtype=np.uint64)[None, :]
    with np.errstate(over="ignore"):
        key = i * np.uint64(n) + j
    h = hash64(seed, 0, key)
    A = ((h >> np.uint64(44)).astype(np.int64) - 524288).astype(np.float64) * 2.0 ** -20
    rows = np.arange(r1 - r0)
    A[rows, np.arange(r0, r1)] = 0.0
    R = np.abs(A).sum(axis=1)          # exact in any order (<= 2^37 units of 2^-20)
    k = (hash64(seed, 1, np.arange(r0, r1, dtype=np.uint64)) >> np.uint64(32)) % np.uint64(kd)
    factor = (17.0 * (1.0 + k.astype(np.float64))) / 16.0
    A[rows, np.arange(r0, r1)] = R * factor
    return A


def gspd(n: int, kappa: float, seed: int = SEED):
    """Full G-SPD matrix, its table and b (small n only)."""
    c = spd_table(n, kappa, seed)
    return gspd_rows(n, c, seed, 0, n), c, rhs(n, seed)


def gdd(n: int, kd: int, seed: int = SEED):
    """Full G-DD matrix and b (small n only)."""
    return gdd_rows(n, kd, seed, 0, n), rhs(n, seed)


def spec(kind: str, n: int, *, kappa: float = 1e3, kd: int = 16, seed: int = SEED) -> dict:
    """Generator spec dict shared by the oracle's Operator(gen=...) and ks_generate."""
    if kind == "spd":
        return {"kind": 0, "n": n, "seed": seed, "kd": 1, "kappa": kappa,
                "table": spd_table(n, kappa, seed)}
    if kind == "dd":
        return {"kind": 1, "n": n, "seed": seed, "kd": kd, "kappa": 0.0, "table": None}
    raise ValueError(kind)


# --- small test matrices (numpy RNG, seeded) --------------------------------

def random_spd(n: int, cond: float, seed: int) -> np.ndarray:
    """Q diag(lambda) Q^T with lambda log-spaced in [1, cond] (Haar Q)."""
    rng = np.random.default_rng(seed)
    Q, R = np.linalg.qr(rng.standard_normal((n, n)))
    Q = Q * np.sign(np.diag(R))
    lam = np.geomspace(1.0, cond, n)
    A = (Q * lam) @ Q.T
    return 0.5 * (A + A.T)


def random_dd(n: int, seed: int, margin: float = 0.5) -> np.ndarray:
    """Dense nonsymmetric strictly row-diagonally-dominant matrix."""
    rng = np.random.default_rng(seed)
    A = rng.uniform(-1.0, 1.0, (n, n))
    np.fill_diagonal(A, 0.0)
    d = np.abs(A).sum(axis=1) * (1.0 + margin) + 1.0
    np.fill_diagonal(A, d * rng.choice([-1.0, 1.0], n))
    return A


def convection_diffusion(n: int = 100, h: float = 0.1) -> np.ndarray:
    """Tridiagonal (-1-h, 2, -1+h), stored dense."""
    A = np.zeros((n, n))
    i = np.arange(n)
    A[i, i] = 2.0
    A[i[1:], i[:-1]] = -1.0 - h
    A[i[:-1], i[1:]] = -1.0 + h
    return A
