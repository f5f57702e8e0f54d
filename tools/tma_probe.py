"""Builds and runs tools/tma_probe.cu (TMA bulk-copy read ceiling) next to the LDG probe."""
import ctypes as C, json, os, subprocess, sys
HERE = os.path.dirname(os.path.abspath(__file__))
so = os.path.join(HERE, "libtmaprobe.so")
subprocess.check_call(["nvcc", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
                       "-Xcompiler", "-fPIC", "-o", so, os.path.join(HERE, "tma_probe.cu")])
L = C.CDLL(so)
L.tma_probe.argtypes = [C.c_double, C.c_int, C.POINTER(C.c_double)]
b = C.c_double()
st = L.tma_probe(float(sys.argv[1]) if len(sys.argv) > 1 else 32.0, 10, C.byref(b))
print(json.dumps({"status": st, "tma_read_gbs": b.value}))
