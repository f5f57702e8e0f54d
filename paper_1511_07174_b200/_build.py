"""Builds libks.so in-tree with nvcc for sm_100a (no JIT, no torch extension cache).

Static cudart (nvcc default), NCCL from the venv's nvidia-nccl wheel -- the same
libnccl.so.2 torch loads, so a communicator borrowed from torch is valid here.
"""
from __future__ import annotations

import concurrent.futures as cf
import importlib.util
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(ROOT, "build", "ks")
LIB = os.path.join(HERE, "libks.so")

SOURCES = ["ks_gemv.cu", "ks_vec.cu", "ks_gen.cu", "ks_persist.cu", "ks_small.cu", "ks_tiny.cu", "ks_multi.cu", "ks_gmres.cu", "ks_gmres_persist.cu", "ks_f32.cu", "ks_alloc.cpp", "ks_ctx.cpp", "ks_solvers.cpp", "ks_abi.cpp"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_root() -> str:
    spec = importlib.util.find_spec("nvidia.nccl")
    if spec is None or not spec.submodule_search_locations:
        raise RuntimeError("nvidia-nccl wheel not found (needed for NCCL headers/lib)")
    return list(spec.submodule_search_locations)[0]


def nvcc() -> str:
    p = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(p):
        raise RuntimeError("nvcc not found")
    return p


def _flags(nroot: str) -> list[str]:
    return ["-O3", "-std=c++17", *ARCH, "-lineinfo", "-Xcompiler", "-fPIC,-Wall",
            "-Xptxas", "-v", "--expt-relaxed-constexpr",
            "-I", os.path.join(ROOT, "include"), "-I", os.path.join(nroot, "include")]


def _compile(src: str, nroot: str) -> tuple[str, str]:
    obj = os.path.join(BUILD, os.path.splitext(src)[0] + ".o")
    path = os.path.join(CSRC, src)
    cmd = [nvcc(), *_flags(nroot), "-c", path, "-o", obj]
    if src.endswith(".cpp"):
        cmd[1:1] = ["-x", "cu"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return obj, r.stderr


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps += [os.path.join(ROOT, "include", "ks.h"), __file__]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    os.makedirs(BUILD, exist_ok=True)
    nroot = nccl_root()
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        results = list(ex.map(lambda s: _compile(s, nroot), SOURCES))
    log = "\n".join(r[1] for r in results)
    with open(os.path.join(BUILD, "ptxas.log"), "w") as f:
        f.write(log)
    if verbose:
        print(log)
    objs = [r[0] for r in results]
    tmp = LIB + f".tmp{os.getpid()}"
    nlib = os.path.join(nroot, "lib")
    cmd = [nvcc(), "-shared", *ARCH, "-o", tmp, *objs, "-L", nlib, "-l:libnccl.so.2",
           "-Xlinker", f"-rpath,{nlib}", "-lpthread"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, LIB)
    return LIB


def build_example() -> str:
    """examples/ks_example: a plain C program against include/ks.h + libks.so."""
    src = os.path.join(ROOT, "examples", "ks_example.c")
    exe = os.path.join(ROOT, "examples", "ks_example")
    if not os.path.exists(src):
        return ""
    subprocess.run(["gcc", "-O2", "-std=c11", "-Wall", "-I", os.path.join(ROOT, "include"), src, "-o", exe,
                    "-L", HERE, "-lks", f"-Wl,-rpath,{HERE}", "-lm"], check=True)
    return exe


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
