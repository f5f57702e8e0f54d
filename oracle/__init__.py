"""CPU oracle for the dense CG / BiCGSTAB hot path (arXiv 1511.07174).

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this module.
The product package ``paper_1511_07174_b200`` never imports it, and this module
never imports the product.  The arithmetic lives in ``ks_oracle.c`` (plain C,
sequential FP64 sums, ``-ffp-contract=off``); this file only marshals arguments
through ctypes and builds the shared object with gcc when it is missing/stale.

Parity status per function: every function below is
pinned by a ``-m "not gpu"`` test in ``tests/test_oracle_*.py``; none is
"parity unpinned".
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ks_oracle.c")
_HDR = os.path.join(_HERE, "ks_oracle.h")
_LIB = os.path.join(_HERE, "liboracle.so")

CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-shared", "-fPIC",
          "-std=c11", "-Wall"]

OK, EARG, EDIM, ENOTSPD, EMAXIT, EBREAKDOWN, ESINGULAR = 0, 1, 2, 3, 4, 5, 6


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (plain C, no CUDA)."""
    stale = (not os.path.exists(_LIB)) or any(
        os.path.getmtime(p) > os.path.getmtime(_LIB) for p in (_SRC, _HDR))
    if force or stale:
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class _Report(C.Structure):
    _fields_ = [("iterations", C.c_int64), ("matvecs", C.c_int64),
                ("converged", C.c_int32), ("breakdown", C.c_int32),
                ("half_step_exit", C.c_int32), ("status", C.c_int32),
                ("relres", C.c_double)]


class _Gen(C.Structure):
    _fields_ = [("kind", C.c_int32), ("n", C.c_int64), ("seed", C.c_uint64),
                ("kd", C.c_int32), ("table", C.POINTER(C.c_double))]


class _Op(C.Structure):
    _fields_ = [("n", C.c_int64), ("A", C.POINTER(C.c_double)), ("lda", C.c_int64),
                ("gen", C.POINTER(_Gen)), ("threads", C.c_int32)]


_lib = None
_D = C.POINTER(C.c_double)


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        i64, i32, u64, dbl = C.c_int64, C.c_int32, C.c_uint64, C.c_double
        L.or_dot.restype = dbl
        L.or_dot.argtypes = [i64, _D, _D]
        L.or_nrm2.restype = dbl
        L.or_nrm2.argtypes = [i64, _D]
        L.or_axpy.argtypes = [i64, dbl, _D, _D]
        L.or_gemv.argtypes = [i64, i64, _D, i64, _D, _D, i32]
        L.or_op_rows.argtypes = [C.POINTER(_Op), i64, i64, _D, _D]
        L.or_cg.restype = C.c_int
        L.or_cg.argtypes = [C.POINTER(_Op), _D, _D, dbl, i64, _D, _D, i64, C.POINTER(_Report),
                            _D, _D, _D, i64]
        L.or_bicgstab.restype = C.c_int
        L.or_bicgstab.argtypes = [C.POINTER(_Op), _D, _D, dbl, i64, _D, _D, i64,
                                  C.POINTER(_Report), _D, _D, i64]
        L.or_ge_solve_ld.restype = C.c_int
        L.or_ge_solve_ld.argtypes = [i64, _D, i64, _D, _D]
        L.or_spd_exact_solve_ld.argtypes = [i64, _D, u64, _D, _D]
        L.or_true_relres_ld.restype = dbl
        L.or_true_relres_ld.argtypes = [C.POINTER(_Op), _D, _D]
        L.or_gemv_t.argtypes = [i64, i64, _D, i64, _D, _D]
        L.or_bicg.restype = C.c_int
        L.or_bicg.argtypes = [i64, _D, i64, _D, _D, dbl, i64, _D, _D, i64, C.POINTER(_Report),
                              _D, _D, _D, _D, i64]
        L.or_gmres.restype = C.c_int
        L.or_gmres.argtypes = [i64, _D, i64, _D, _D, dbl, i64, i64, _D, _D, i64, C.POINTER(_Report)]
        _F = C.POINTER(C.c_float)
        flt = C.c_float
        L.or_cg_f32.restype = C.c_int
        L.or_cg_f32.argtypes = [i64, _F, i64, _F, flt, i64, _F, _F, i64, C.POINTER(_Report)]
        L.or_bicgstab_f32.restype = C.c_int
        L.or_bicgstab_f32.argtypes = [i64, _F, i64, _F, flt, i64, _F, _F, i64, C.POINTER(_Report)]
        L.or_hash.restype = u64
        L.or_hash.argtypes = [u64, u64, u64]
        L.or_gen_rows.argtypes = [C.POINTER(_Gen), i64, i64, _D, i64]
        L.or_gen_rows_par.argtypes = [C.POINTER(_Gen), i64, i64, _D, i64, i32]
        L.or_gen_rhs.argtypes = [i64, u64, _D]
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(_D)


def _vec(a, n=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    if n is not None and a.shape != (n,):
        raise ValueError(f"expected shape ({n},), got {a.shape}")
    return a


@dataclass
class Report:
    iterations: int
    matvecs: int
    converged: bool
    breakdown: bool
    half_step_exit: bool
    status: int
    relres: float


class Operator:
    """A stored row-major matrix, or a generator spec expanded row by row."""

    def __init__(self, A=None, *, gen: dict | None = None, threads: int = 1):
        self._keep = []
        if A is not None:
            A = np.ascontiguousarray(A, dtype=np.float64)
            if A.ndim != 2 or A.shape[0] != A.shape[1]:
                raise ValueError("A must be square")
            self.n = A.shape[0]
            self._keep.append(A)
            self._op = _Op(self.n, _p(A), A.shape[1], None, threads)
        else:
            g = gen
            self.n = int(g["n"])
            table = g.get("table")
            if table is not None:
                table = _vec(table, self.n)
                self._keep.append(table)
            self._gen = _Gen(int(g["kind"]), self.n, int(g["seed"]), int(g.get("kd", 1)),
                             _p(table))
            self._op = _Op(self.n, None, 0, C.pointer(self._gen), threads)

    @property
    def ref(self):
        return C.byref(self._op)

    def rows(self, r0: int, nrows: int, x) -> np.ndarray:
        """y[r] = sum_j a_{r0+r, j} x_j, sequential per row."""
        x = _vec(x, self.n)
        y = np.empty(nrows)
        lib().or_op_rows(self.ref, r0, nrows, _p(x), _p(y))
        return y

    def apply(self, x) -> np.ndarray:
        return self.rows(0, self.n, x)


def _as_op(A) -> Operator:
    return A if isinstance(A, Operator) else Operator(A)


def dot(x, y) -> float:
    x, y = _vec(x), _vec(y)
    return lib().or_dot(x.size, _p(x), _p(y))


def nrm2(x) -> float:
    x = _vec(x)
    return lib().or_nrm2(x.size, _p(x))


def axpy(alpha, x, y) -> np.ndarray:
    x, y = _vec(x), _vec(y).copy()
    lib().or_axpy(x.size, float(alpha), _p(x), _p(y))
    return y


def gemv(A, x, threads: int = 1) -> np.ndarray:
    A = np.ascontiguousarray(A, dtype=np.float64)
    x = _vec(x, A.shape[1])
    y = np.empty(A.shape[0])
    lib().or_gemv(A.shape[0], A.shape[1], _p(A), A.shape[1], _p(x), _p(y), threads)
    return y


def _rep(r: _Report) -> Report:
    return Report(int(r.iterations), int(r.matvecs), bool(r.converged), bool(r.breakdown),
                  bool(r.half_step_exit), int(r.status), float(r.relres))


def cg(A, b, x0=None, tol=1e-8, maxit=None, trace: int = 0):
    """SURVEY.md sec.8(c).3.  Returns (x, hist, report[, trace dict])."""
    op = _as_op(A)
    n = op.n
    b = _vec(b, n)
    x0 = None if x0 is None else _vec(x0, n)
    maxit = 10 * n if maxit is None else int(maxit)
    x = np.empty(n)
    hist = np.zeros(max(maxit, 1))
    rep = _Report()
    tx = tr = tp = None
    if trace:
        tx, tr, tp = (np.zeros((trace, n)) for _ in range(3))
    lib().or_cg(op.ref, _p(b), _p(x0), float(tol), maxit, _p(x), _p(hist), maxit,
                C.byref(rep), _p(tx), _p(tr), _p(tp), trace)
    R = _rep(rep)
    out = (x, hist[:min(R.iterations, maxit)].copy(), R)
    if trace:
        return out + ({"x": tx, "r": tr, "p": tp},)
    return out


def bicgstab(A, b, x0=None, tol=1e-8, maxit=None, trace: int = 0):
    """SURVEY.md sec.8(c).4.  Returns (x, hist, report[, trace dict])."""
    op = _as_op(A)
    n = op.n
    b = _vec(b, n)
    x0 = None if x0 is None else _vec(x0, n)
    maxit = 10 * n if maxit is None else int(maxit)
    x = np.empty(n)
    hist = np.zeros(max(maxit, 1))
    rep = _Report()
    ts = tr = None
    if trace:
        ts, tr = np.zeros((trace, n)), np.zeros((trace, n))
    lib().or_bicgstab(op.ref, _p(b), _p(x0), float(tol), maxit, _p(x), _p(hist), maxit,
                      C.byref(rep), _p(ts), _p(tr), trace)
    R = _rep(rep)
    out = (x, hist[:min(R.iterations, maxit)].copy(), R)
    if trace:
        return out + ({"s": ts, "r": tr},)
    return out


def cg_multi(A, B, X0=None, tol=1e-8, maxit=None):
    """Multi-RHS CG (SURVEY.md sec.8(f) "multi-RHS"; reading Q30): column k
    of the n x nrhs block B is solved by the CG of sec.8(c).3 on (A, B[:, k]) with its
    own scalars and stopping test -- exactly ``cg`` per column (the GPU shares the
    passes over A between the columns; the recurrences are independent).  Returns
    (X n x nrhs, [hist_k], [report_k])."""
    B = np.asarray(B, dtype=np.float64)
    if B.ndim != 2:
        raise ValueError("B must be n x nrhs")
    X = np.empty_like(B)
    hs, reps = [], []
    for k in range(B.shape[1]):
        x0 = None if X0 is None else np.asarray(X0, dtype=np.float64)[:, k]
        x, h, r = cg(A, B[:, k], x0=x0, tol=tol, maxit=maxit)
        X[:, k] = x
        hs.append(h)
        reps.append(r)
    return X, hs, reps


def bicgstab_multi(A, B, X0=None, tol=1e-8, maxit=None):
    """Multi-RHS BiCGSTAB (reading Q30 applied to SURVEY.md sec.8(c).4):
    column k of B solved by ``bicgstab`` on (A, B[:, k]) -- the recurrences are
    independent; the GPU shares the two GEMMs of each iteration between the columns.
    Returns (X n x nrhs, [hist_k], [report_k])."""
    B = np.asarray(B, dtype=np.float64)
    if B.ndim != 2:
        raise ValueError("B must be n x nrhs")
    X = np.empty_like(B)
    hs, reps = [], []
    for k in range(B.shape[1]):
        x0 = None if X0 is None else np.asarray(X0, dtype=np.float64)[:, k]
        x, h, r = bicgstab(A, B[:, k], x0=x0, tol=tol, maxit=maxit)
        X[:, k] = x
        hs.append(h)
        reps.append(r)
    return X, hs, reps


def gemv_t(A, x) -> np.ndarray:
    """y = A^T x for row-major A (sequential sums over rows)."""
    A = np.ascontiguousarray(A, dtype=np.float64)
    x = _vec(x, A.shape[0])
    y = np.empty(A.shape[1])
    lib().or_gemv_t(A.shape[0], A.shape[1], _p(A), A.shape[1], _p(x), _p(y))
    return y


def bicg(A, b, x0=None, tol=1e-8, maxit=None, trace: int = 0):
    """BiCG.  Returns (x, hist, report[, trace dict r, rt, p, pt])."""
    A = np.ascontiguousarray(A, dtype=np.float64)
    n = A.shape[0]
    b = _vec(b, n)
    x0 = None if x0 is None else _vec(x0, n)
    maxit = 10 * n if maxit is None else int(maxit)
    x = np.empty(n)
    hist = np.zeros(max(maxit, 1))
    rep = _Report()
    tr = [None] * 4
    if trace:
        tr = [np.zeros((trace, n)) for _ in range(4)]
    lib().or_bicg(n, _p(A), n, _p(b), _p(x0), float(tol), maxit, _p(x), _p(hist), maxit,
                  C.byref(rep), *(_p(t) for t in tr), trace)
    R = _rep(rep)
    out = (x, hist[:min(R.iterations, maxit)].copy(), R)
    if trace:
        return out + (dict(zip(("r", "rt", "p", "pt"), tr)),)
    return out


def gmres(A, b, x0=None, tol=1e-8, restart=30, maxit=None):
    """Restarted GMRES(m) with MGS Arnoldi.  hist = implicit residuals."""
    A = np.ascontiguousarray(A, dtype=np.float64)
    n = A.shape[0]
    b = _vec(b, n)
    x0 = None if x0 is None else _vec(x0, n)
    maxit = 10 * n if maxit is None else int(maxit)
    x = np.empty(n)
    hist = np.zeros(max(maxit, 1))
    rep = _Report()
    lib().or_gmres(n, _p(A), n, _p(b), _p(x0), float(tol), int(restart), maxit, _p(x), _p(hist),
                   maxit, C.byref(rep))
    R = _rep(rep)
    return x, hist[:min(R.iterations, maxit)].copy(), R


def _solve_f32(fn, A, b, tol, maxit):
    A = np.ascontiguousarray(A, dtype=np.float32)
    n = A.shape[0]
    b = np.ascontiguousarray(b, dtype=np.float32)
    maxit = 10 * n if maxit is None else int(maxit)
    x = np.empty(n, dtype=np.float32)
    hist = np.zeros(max(maxit, 1), dtype=np.float32)
    rep = _Report()
    F = C.POINTER(C.c_float)
    fn(n, A.ctypes.data_as(F), n, b.ctypes.data_as(F), C.c_float(tol), maxit, x.ctypes.data_as(F),
       hist.ctypes.data_as(F), maxit, C.byref(rep))
    R = _rep(rep)
    return x, hist[:min(R.iterations, maxit)].copy(), R


def cg_f32(A, b, tol=1e-5, maxit=None):
    """NEXT-4: CG in binary32 (A, b rounded to float by the caller or here)."""
    return _solve_f32(lib().or_cg_f32, A, b, tol, maxit)


def bicgstab_f32(A, b, tol=1e-5, maxit=None):
    """NEXT-4: BiCGSTAB in binary32."""
    return _solve_f32(lib().or_bicgstab_f32, A, b, tol, maxit)


def ge_solve_ld(A, b) -> np.ndarray:
    """Long-double Gaussian elimination with partial pivoting (pin P5)."""
    A = np.ascontiguousarray(A, dtype=np.float64)
    n = A.shape[0]
    b = _vec(b, n)
    x = np.empty(n)
    st = lib().or_ge_solve_ld(n, _p(A), n, _p(b), _p(x))
    if st != OK:
        raise np.linalg.LinAlgError(f"or_ge_solve_ld status {st}")
    return x


def spd_exact_solve_ld(table, seed: int, b) -> np.ndarray:
    """Closed-form solution of the G-SPD system (pin P6)."""
    table = _vec(table)
    n = table.size
    b = _vec(b, n)
    x = np.empty(n)
    lib().or_spd_exact_solve_ld(n, _p(table), int(seed), _p(b), _p(x))
    return x


def true_relres_ld(A, b, x) -> float:
    op = _as_op(A)
    b, x = _vec(b, op.n), _vec(x, op.n)
    return lib().or_true_relres_ld(op.ref, _p(b), _p(x))


def hash64(seed: int, stream: int, key: int) -> int:
    return int(lib().or_hash(seed, stream, key))


def gen_rows(gen: dict, r0: int, nrows: int, threads: int = 1) -> np.ndarray:
    """Rows [r0, r0 + nrows) of the generated matrix (bitwise the same for any
    thread count: rows are expanded independently)."""
    n = int(gen["n"])
    op = Operator(gen=gen)
    A = np.empty((nrows, n))
    if threads > 1:
        lib().or_gen_rows_par(op._op.gen, r0, nrows, _p(A), n, threads)
    else:
        lib().or_gen_rows(op._op.gen, r0, nrows, _p(A), n)
    return A


def gen_rhs(n: int, seed: int) -> np.ndarray:
    b = np.empty(n)
    lib().or_gen_rhs(n, int(seed), _p(b))
    return b
