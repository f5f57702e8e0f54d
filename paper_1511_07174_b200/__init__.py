"""B200-native dense Krylov hot path of arXiv 1511.07174 (CUPLSS): FP64 CG and
BiCGSTAB on dense row-major matrices, row-block sharded over GPUs.

This module is the thin Python binding of the C ABI in ``include/ks.h``: it only
marshals arguments (numpy arrays, torch tensors, raw pointers) through ctypes.
Every step of the method runs in ``libks.so`` (hand-written sm_100a kernels +
NCCL).  There is no CPU fallback: if ``libks.so`` is missing, import fails.

    import paper_1511_07174_b200 as ks
    ctx = ks.Context(n, ngpus=1)
    b = ctx.generate("spd", table=synth.spd_table(n, 1e4), seed=...)
    x, hist, rep = ctx.cg(b, tol=1e-10)
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libks.so")

KS_OK, KS_EARG, KS_EDIM, KS_ENOTSPD, KS_EMAXIT, KS_EBREAKDOWN = 0, 1, 2, 3, 4, 5
KS_ECUDA, KS_ENCCL, KS_ENOMEM, KS_ESTATE = 6, 7, 8, 9
DTYPES = {"f64": 0, "float64": 0, "f32": 1, "float32": 1}
STATUS_NAMES = {0: "OK", 1: "EARG", 2: "EDIM", 3: "ENOTSPD", 4: "EMAXIT", 5: "EBREAKDOWN",
                6: "ECUDA", 7: "ENCCL", 8: "ENOMEM", 9: "ESTATE"}
OPTIONS = {"true_residual": 0, "profile_gemv": 1, "poll_batch": 2, "gemv_rows": 3,
           "gemv_split": 4, "gemv_kernel": 5, "use_graphs": 6, "fused_comm": 7,
           "persistent": 8, "gemv_unroll": 9, "persist_grid": 10,
           "gemvt_shape": 11, "small": 12, "join_timeout_ms": 13,
           "tiny": 14, "jitter": 15, "ll_xchg": 16}
EXPORTS = ["ks_create", "ks_create_on", "ks_create_rank", "ks_destroy", "ks_row_range", "ks_load_rows",
           "ks_generate", "ks_matvec", "ks_matvec_t", "ks_time_matvec", "ks_cg", "ks_bicgstab",
           "ks_bicg", "ks_gmres", "ks_cg_multi", "ks_bicgstab_multi",
           "ks_set_option", "ks_get_option", "ks_info", "ks_check_guards", "ks_last_error", "ks_version"]


class KsError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class _Report(C.Structure):
    _fields_ = [("iterations", C.c_int64), ("matvecs", C.c_int64), ("converged", C.c_int32),
                ("breakdown", C.c_int32), ("half_step_exit", C.c_int32), ("status", C.c_int32),
                ("relres", C.c_double), ("true_relres", C.c_double),
                ("seconds_loop", C.c_double), ("seconds_total", C.c_double),
                ("seconds_gemv", C.c_double), ("gemv_launches", C.c_int64),
                ("kernel_launches", C.c_int64)]


class _GenSpec(C.Structure):
    _fields_ = [("kind", C.c_int32), ("seed", C.c_uint64), ("kappa", C.c_double),
                ("kd", C.c_int32), ("spd_table", C.c_void_p)]


@dataclass
class Report:
    iterations: int
    matvecs: int
    converged: bool
    breakdown: bool
    half_step_exit: bool
    status: int
    relres: float
    true_relres: float
    seconds_loop: float
    seconds_total: float
    seconds_gemv: float
    gemv_launches: int
    kernel_launches: int

    @property
    def status_name(self) -> str:
        return STATUS_NAMES.get(self.status, str(self.status))


_lib = None


def lib():
    """Loads libks.so (fails loudly when it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        vp, i64, i32, dbl = C.c_void_p, C.c_int64, C.c_int32, C.c_double
        pp = C.POINTER(C.c_void_p)
        sig = {
            "ks_create": [pp, i64, C.c_int, i32],
            "ks_create_on": [pp, i64, C.c_int, i32, C.POINTER(i32)],
            "ks_create_rank": [pp, i64, C.c_int, i32, i32, vp, i32, vp],
            "ks_destroy": [vp],
            "ks_row_range": [vp, i32, C.POINTER(i64), C.POINTER(i64)],
            "ks_load_rows": [vp, i64, i64, vp, i64],
            "ks_generate": [vp, C.POINTER(_GenSpec), vp],
            "ks_matvec": [vp, vp, vp],
            "ks_matvec_t": [vp, vp, vp],
            "ks_bicg": [vp, vp, vp, dbl, i64, vp, vp, i64, C.POINTER(_Report)],
            "ks_gmres": [vp, vp, vp, dbl, i32, i64, vp, vp, i64, C.POINTER(_Report)],
            "ks_time_matvec": [vp, i32, C.POINTER(dbl)],
            "ks_cg": [vp, vp, vp, dbl, i64, vp, vp, i64, C.POINTER(_Report)],
            "ks_bicgstab": [vp, vp, vp, dbl, i64, vp, vp, i64, C.POINTER(_Report)],
            "ks_cg_multi": [vp, i32, vp, vp, dbl, i64, vp, vp, i64, C.POINTER(_Report)],
            "ks_bicgstab_multi": [vp, i32, vp, vp, dbl, i64, vp, vp, i64, C.POINTER(_Report)],
            "ks_set_option": [vp, C.c_int, i64],
            "ks_get_option": [vp, C.c_int, C.POINTER(i64)],
            "ks_info": [vp, C.POINTER(i32), C.POINTER(i32), C.POINTER(i64), C.POINTER(i64)],
            "ks_check_guards": [vp, C.POINTER(i64)],
        }
        for name, args in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = C.c_int
        L.ks_last_error.argtypes = [vp]
        L.ks_last_error.restype = C.c_char_p
        L.ks_version.argtypes = []
        L.ks_version.restype = C.c_char_p
        _lib = L
    return _lib


def version() -> str:
    return lib().ks_version().decode()


def _ptr(a):
    """Raw pointer of a numpy array or torch tensor (host or device); None -> NULL."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    if isinstance(a, int):
        return a
    raise TypeError(f"unsupported buffer type {type(a)}")


def _f64(a, n: int, name: str):
    if a is None:
        return None
    if hasattr(a, "data_ptr") and not isinstance(a, np.ndarray):
        import torch
        if a.dtype != torch.float64 or a.numel() != n or not a.is_contiguous():
            raise ValueError(f"{name}: need a contiguous float64 tensor of {n} elements")
        return a
    a = np.ascontiguousarray(a, dtype=np.float64)
    if a.shape != (n,):
        raise ValueError(f"{name}: expected shape ({n},), got {a.shape}")
    return a


def _out64(a, n: int | None, name: str):
    """An OUTPUT buffer: written in place by the library, so it must already be a
    contiguous 1-D float64 array / tensor (a converted copy would leave the
    caller's buffer unwritten; a wrong dtype or stride would overflow it)."""
    if a is None:
        return None
    if hasattr(a, "data_ptr") and not isinstance(a, np.ndarray):
        import torch
        if a.dtype != torch.float64 or a.dim() != 1 or not a.is_contiguous() or \
                (n is not None and a.numel() != n):
            raise ValueError(f"{name}: need a contiguous 1-D float64 tensor"
                             + (f" of {n} elements" if n is not None else ""))
        return a
    if not isinstance(a, np.ndarray) or a.dtype != np.float64 or a.ndim != 1 or \
            not a.flags["C_CONTIGUOUS"] or not a.flags["WRITEABLE"] or (n is not None and a.shape[0] != n):
        raise ValueError(f"{name}: need a writeable contiguous 1-D float64 array"
                         + (f" of {n} elements" if n is not None else ""))
    return a


class Context:
    """Opaque solver context: A resident in HBM, row-block sharded."""

    def __init__(self, n: int, ngpus: int = 1, *, dtype: str = "f64", devices=None, _handle=None):
        """ngpus ranks on GPUs 0..ngpus-1, or rank g on devices[g] (ks_create_on: a
        device may repeat -- its ranks split its SMs; for validating P > 1 schedules
        on fewer GPUs)."""
        self._h = C.c_void_p()
        self.dtype = "f32" if DTYPES[dtype] == 1 else "f64"
        if _handle is not None:
            self._h = _handle
        elif devices is not None:
            devs = (C.c_int32 * len(devices))(*[int(d) for d in devices])
            self._check(lib().ks_create_on(C.byref(self._h), int(n), DTYPES[dtype], len(devices), devs))
        else:
            self._check(lib().ks_create(C.byref(self._h), int(n), DTYPES[dtype], int(ngpus)))
        lg, nr, nn, ld = C.c_int32(), C.c_int32(), C.c_int64(), C.c_int64()
        self._check(lib().ks_info(self._h, C.byref(lg), C.byref(nr), C.byref(nn), C.byref(ld)))
        self.n, self.nranks, self.local_gpus, self.ld = nn.value, nr.value, lg.value, ld.value

    @classmethod
    def from_rank(cls, n: int, rank: int, nranks: int, nccl_comm: int | None, device: int,
                  stream: int | None = None, dtype: str = "f64") -> "Context":
        h = C.c_void_p()
        st = lib().ks_create_rank(C.byref(h), int(n), DTYPES[dtype], int(rank), int(nranks), nccl_comm,
                                  int(device), stream)
        if st != KS_OK:
            raise KsError(st, lib().ks_last_error(None).decode())
        return cls(n, dtype=dtype, _handle=h)

    @classmethod
    def from_process_group(cls, n: int, group=None, stream=None, dtype: str = "f64") -> "Context":
        """One rank per process (torchrun): borrows torch's NCCL communicator and
        the current CUDA stream.  torch is only the plumbing here."""
        import torch
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        dev = torch.cuda.current_device()
        s = stream if stream is not None else torch.cuda.current_stream()
        comm = None
        if world > 1:
            pg = group if group is not None else dist.group.WORLD
            t = torch.zeros(1, device=f"cuda:{dev}")
            dist.all_reduce(t, group=pg)           # makes sure the communicator exists
            torch.cuda.synchronize()
            comm = pg._get_backend(torch.device("cuda"))._comm_ptr()
        return cls.from_rank(n, rank, world, comm, dev, s.cuda_stream, dtype=dtype)

    # -- plumbing ---------------------------------------------------------------
    def _check(self, st: int, ok=(KS_OK,)):
        if st not in ok:
            raise KsError(st, lib().ks_last_error(self._h).decode())
        return st

    def close(self):
        if self._h:
            lib().ks_destroy(self._h)
            self._h = C.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_option(self, name: str, value: int):
        self._check(lib().ks_set_option(self._h, OPTIONS[name], int(value)))

    def check_guards(self) -> int:
        """Corrupted guard zones (out-of-bounds writes) with KS_GUARD=1; -1 otherwise."""
        v = C.c_int64()
        self._check(lib().ks_check_guards(self._h, C.byref(v)))
        return v.value

    def get_option(self, name: str) -> int:
        v = C.c_int64()
        self._check(lib().ks_get_option(self._h, OPTIONS[name], C.byref(v)))
        return v.value

    def row_range(self, shard: int) -> tuple[int, int]:
        b, e = C.c_int64(), C.c_int64()
        self._check(lib().ks_row_range(self._h, int(shard), C.byref(b), C.byref(e)))
        return b.value, e.value

    # -- inputs -----------------------------------------------------------------
    def load_rows(self, A, row_begin: int = 0):
        """Rows [row_begin, row_begin + A.shape[0]) of the row-major matrix."""
        A = np.ascontiguousarray(A, dtype=np.float64)
        if A.ndim != 2 or A.shape[1] != self.n:
            raise ValueError(f"A must be (rows, {self.n})")
        self._check(lib().ks_load_rows(self._h, int(row_begin), A.shape[0], _ptr(A), A.shape[1]))

    def generate(self, kind: str, *, seed: int, table=None, kd: int = 16, kappa: float = 0.0,
                 want_b: bool = True):
        """Expands G-SPD ('spd', needs the circulant `table`) or G-DD ('dd') on the
        device; returns b (numpy) when want_b."""
        spec = _GenSpec()
        spec.kind = {"spd": 0, "dd": 1}[kind]
        spec.seed = int(seed)
        spec.kappa = float(kappa)
        spec.kd = int(kd)
        tab = None
        if kind == "spd":
            tab = np.ascontiguousarray(table, dtype=np.float64)
            if tab.shape != (self.n,):
                raise ValueError("table must have n entries")
            spec.spd_table = tab.ctypes.data
        b = np.empty(self.n) if want_b else None
        self._check(lib().ks_generate(self._h, C.byref(spec), _ptr(b)))
        return b

    # -- compute ----------------------------------------------------------------
    def matvec(self, x, out=None):
        x = _f64(x, self.n, "x")
        y = np.empty(self.n) if out is None else _out64(out, self.n, "out")
        self._check(lib().ks_matvec(self._h, _ptr(x), _ptr(y)))
        return y

    def matvec_t(self, x, out=None):
        """y = A^T x (the transposed GEMV of BiCG)."""
        x = _f64(x, self.n, "x")
        y = np.empty(self.n) if out is None else _out64(out, self.n, "out")
        self._check(lib().ks_matvec_t(self._h, _ptr(x), _ptr(y)))
        return y

    def time_matvec(self, reps: int = 20) -> float:
        s = C.c_double()
        self._check(lib().ks_time_matvec(self._h, int(reps), C.byref(s)))
        return s.value

    def _solve(self, fn, b, x0, tol, maxit, out, hist, hist_cap):
        b = _f64(b, self.n, "b")
        x0 = _f64(x0, self.n, "x0")
        maxit = 10 * self.n if maxit is None else int(maxit)
        x = np.empty(self.n) if out is None else _out64(out, self.n, "out")
        if hist is True:
            hist = np.zeros(max(1, min(maxit, hist_cap)))
        elif hist is False or hist is None:
            hist = None
        else:
            hist = _out64(hist, None, "hist")
        cap = 0 if hist is None else (hist.shape[0] if isinstance(hist, np.ndarray) else hist.numel())
        rep = _Report()
        st = fn(self._h, _ptr(b), _ptr(x0), float(tol), maxit, _ptr(x), _ptr(hist), cap,
                C.byref(rep))
        self._check(st, ok=(KS_OK, KS_EMAXIT, KS_ENOTSPD, KS_EBREAKDOWN))
        R = Report(int(rep.iterations), int(rep.matvecs), bool(rep.converged), bool(rep.breakdown),
                   bool(rep.half_step_exit), int(rep.status), float(rep.relres),
                   float(rep.true_relres), float(rep.seconds_loop), float(rep.seconds_total),
                   float(rep.seconds_gemv), int(rep.gemv_launches), int(rep.kernel_launches))
        if isinstance(hist, np.ndarray):
            hist = hist[: min(R.iterations, cap)].copy()
        return x, hist, R

    def cg(self, b, x0=None, tol: float = 1e-8, maxit: int | None = None, *, out=None,
           hist=True, hist_cap: int = 1 << 20):
        """CG.  Returns (x, hist, Report)."""
        return self._solve(lib().ks_cg, b, x0, tol, maxit, out, hist, hist_cap)

    def bicg(self, b, x0=None, tol: float = 1e-8, maxit: int | None = None, *, out=None,
             hist=True, hist_cap: int = 1 << 20):
        """BiCG (NEXT-3).  Returns (x, hist, Report)."""
        return self._solve(lib().ks_bicg, b, x0, tol, maxit, out, hist, hist_cap)

    def gmres(self, b, x0=None, tol: float = 1e-8, restart: int = 30, maxit: int | None = None, *,
              out=None, hist=True, hist_cap: int = 1 << 20):
        """Restarted GMRES(m) (NEXT-3).  Returns (x, hist, Report)."""
        r = int(restart)
        fn = lambda h, b_, x0_, tol_, mx, x_, hi, cap, rep: lib().ks_gmres(h, b_, x0_, tol_, r, mx, x_, hi, cap, rep)
        return self._solve(fn, b, x0, tol, maxit, out, hist, hist_cap)

    def cg_multi(self, B, X0=None, tol: float = 1e-8, maxit: int | None = None, *, hist=True,
                 hist_cap: int = 1 << 16):
        """Multi-RHS CG (ks_cg_multi): B is n x nrhs (1 <= nrhs <= 8), column k one
        right-hand side; independent CG recurrences sharing every pass over A.
        Returns (X n x nrhs, [hist_k], [Report_k])."""
        return self._multi(lib().ks_cg_multi, B, X0, tol, maxit, hist, hist_cap)

    def bicgstab_multi(self, B, X0=None, tol: float = 1e-8, maxit: int | None = None, *, hist=True,
                       hist_cap: int = 1 << 16):
        """Multi-RHS BiCGSTAB (ks_bicgstab_multi, one GPU): as cg_multi."""
        return self._multi(lib().ks_bicgstab_multi, B, X0, tol, maxit, hist, hist_cap)

    def _multi(self, fn, B, X0, tol, maxit, hist, hist_cap):
        B = np.asfortranarray(B, dtype=np.float64)
        if B.ndim != 2 or B.shape[0] != self.n:
            raise ValueError(f"B must be ({self.n}, nrhs)")
        k = B.shape[1]
        X0 = None if X0 is None else np.asfortranarray(X0, dtype=np.float64)
        if X0 is not None and X0.shape != B.shape:
            raise ValueError("X0 must have the shape of B")
        maxit = 10 * self.n if maxit is None else int(maxit)
        X = np.empty((self.n, k), order="F")
        cap = max(1, min(maxit, hist_cap)) if hist else 0
        H = np.zeros((cap, k), order="F") if hist else None
        reps = (_Report * k)()
        st = fn(self._h, k, _ptr(B), _ptr(X0), float(tol), maxit, _ptr(X), _ptr(H), cap, reps)
        self._check(st, ok=(KS_OK, KS_EMAXIT, KS_ENOTSPD, KS_EBREAKDOWN))
        R = [Report(int(q.iterations), int(q.matvecs), bool(q.converged), bool(q.breakdown),
                    bool(q.half_step_exit), int(q.status), float(q.relres), float(q.true_relres),
                    float(q.seconds_loop), float(q.seconds_total), float(q.seconds_gemv),
                    int(q.gemv_launches), int(q.kernel_launches)) for q in reps]
        hs = [H[: min(r.iterations, cap), j].copy() for j, r in enumerate(R)] if hist else [None] * k
        return X, hs, R

    def bicgstab(self, b, x0=None, tol: float = 1e-8, maxit: int | None = None, *, out=None,
                 hist=True, hist_cap: int = 1 << 20):
        """BiCGSTAB.  Returns (x, hist, Report)."""
        return self._solve(lib().ks_bicgstab, b, x0, tol, maxit, out, hist, hist_cap)


def cg(A, b, x0=None, tol=1e-8, maxit=None, ngpus: int = 1):
    """One-shot convenience: loads the dense matrix and runs CG."""
    A = np.ascontiguousarray(A, dtype=np.float64)
    with Context(A.shape[0], ngpus) as ctx:
        ctx.load_rows(A)
        return ctx.cg(b, x0, tol, maxit)


def bicgstab(A, b, x0=None, tol=1e-8, maxit=None, ngpus: int = 1):
    A = np.ascontiguousarray(A, dtype=np.float64)
    with Context(A.shape[0], ngpus) as ctx:
        ctx.load_rows(A)
        return ctx.bicgstab(b, x0, tol, maxit)


def partition(n: int, P: int) -> list[tuple[int, int]]:
    """Row ranges of the 1-D row-block partition (mirrors ks_row_range; host logic)."""
    q, rem = divmod(n, P)
    out = []
    for g in range(P):
        b = g * q + min(g, rem)
        out.append((b, b + q + (1 if g < rem else 0)))
    return out
