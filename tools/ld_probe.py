"""Builds and runs tools/ld_probe.cu (LDG cache-qualifier / L2 prefetch variants)."""
import ctypes as C, os, subprocess, sys
HERE = os.path.dirname(os.path.abspath(__file__))
so = os.path.join(HERE, "libldprobe.so")
subprocess.check_call(["nvcc", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
                       "-Xcompiler", "-fPIC", "-o", so, os.path.join(HERE, "ld_probe.cu")])
L = C.CDLL(so)
L.ld_probe.argtypes = [C.c_double, C.c_int]
sys.exit(L.ld_probe(float(sys.argv[1]) if len(sys.argv) > 1 else 32.0, 10))
