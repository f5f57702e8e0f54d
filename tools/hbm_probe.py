"""Builds and runs tools/hbm_probe.cu: best read-only and copy bandwidth on GPU 0."""
import ctypes as C, json, os, subprocess, sys
HERE = os.path.dirname(os.path.abspath(__file__))
so = os.path.join(HERE, "libprobe.so")
subprocess.check_call(["nvcc", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
                       "-Xcompiler", "-fPIC", "-o", so, os.path.join(HERE, "hbm_probe.cu")])
L = C.CDLL(so)
L.probe.argtypes = [C.c_double, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_int)]
r, c, cfg = C.c_double(), C.c_double(), C.c_int()
st = L.probe(float(sys.argv[1]) if len(sys.argv) > 1 else 32.0, 10, C.byref(r), C.byref(c), C.byref(cfg))
res = {"status": st, "read_gbs": r.value, "copy_gbs": c.value, "best_cfg": cfg.value}
print(json.dumps(res))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/hbm_probe.json", "w"))
