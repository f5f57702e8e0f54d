"""CPU-side checks of the boundary: libks.so loads, exports every symbol that
include/ks.h declares, and the host-only paths behave (no compute without a GPU)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_1511_07174_b200 as ks

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "ks.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ks_[a-z_]+)\s*\(", src)))


def test_header_declares_the_survey_entry_points():
    d = _declared()
    for name in ["ks_create", "ks_create_rank", "ks_destroy", "ks_row_range", "ks_load_rows",
                 "ks_generate", "ks_matvec", "ks_time_matvec", "ks_cg", "ks_bicgstab",
                 "ks_last_error"]:
        assert name in d


def test_library_exports_every_declared_symbol():
    L = ks.lib()
    for name in _declared():
        assert hasattr(L, name), name
    assert sorted(ks.EXPORTS) == _declared()


def test_library_links_venv_nccl_and_is_sm100a():
    import subprocess
    out = subprocess.run(["ldd", ks.LIB_PATH], capture_output=True, text=True).stdout
    assert "nvidia/nccl/lib/libnccl.so.2" in out
    sass = subprocess.run(["cuobjdump", "--list-elf", ks.LIB_PATH], capture_output=True,
                          text=True).stdout
    assert "sm_100a" in sass


def test_version_and_errors_without_gpu():
    assert "sm_100a" in ks.version()
    h = C.c_void_p()
    # no device here (or wrong args) -> an error code, never a crash
    st = ks.lib().ks_create(C.byref(h), 1024, 0, 0)
    assert st == ks.KS_EARG
    assert b"ngpus" in ks.lib().ks_last_error(None)
    st = ks.lib().ks_create(C.byref(h), 0, 0, 1)
    assert st == ks.KS_EDIM
    st = ks.lib().ks_create(C.byref(h), 16, 7, 1)
    assert st == ks.KS_EARG
    st = ks.lib().ks_create_rank(C.byref(h), 16, 0, 2, 2, None, 0, None)
    assert st == ks.KS_EARG
    st = ks.lib().ks_create_on(C.byref(h), 16, 0, 2, None)
    assert st == ks.KS_EARG
    devs = (C.c_int32 * 2)(0, 0)
    st = ks.lib().ks_create_on(C.byref(h), 16, 0, 2, devs)     # no device 0 here
    assert st == ks.KS_EARG and b"not a device" in ks.lib().ks_last_error(None)
    st = ks.lib().ks_create_on(C.byref(h), 16, 0, 17, devs)
    assert st == ks.KS_EARG
    assert ks.lib().ks_destroy(None) == ks.KS_OK


@pytest.mark.parametrize("n,P", [(1, 1), (10, 3), (65536, 8), (1023, 4), (7, 7)])
def test_partition_covers_rows(n, P):
    parts = ks.partition(n, P)
    assert parts[0][0] == 0 and parts[-1][1] == n
    assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
    sizes = [e - b for b, e in parts]
    assert max(sizes) - min(sizes) <= 1
    assert sizes == sorted(sizes, reverse=True)   # first n mod P shards get the extra row


def test_product_does_not_import_oracle():
    """The product package must not reach the oracle (no CPU fallback)."""
    for root, _, files in os.walk(os.path.join(ROOT, "paper_1511_07174_b200")):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".h", ".cuh")):
                txt = open(os.path.join(root, f)).read()
                assert "import oracle" not in txt and "ks_oracle" not in txt, f
                assert "from oracle" not in txt, f


def test_c_example_links_against_the_abi():
    """examples/ks_example.c builds against include/ks.h + libks.so with plain gcc."""
    from paper_1511_07174_b200 import _build
    exe = _build.build_example()
    assert os.path.exists(exe)


def test_output_buffers_are_validated_not_copied():
    """out= and hist= are written in place by the library: a wrong dtype, a strided
    view or a read-only array is rejected instead of silently copied (the caller's
    buffer would never be written) or overflowed."""
    import pytest
    from paper_1511_07174_b200 import _out64
    ok = np.zeros(8)
    assert _out64(ok, 8, "x") is ok
    assert _out64(np.zeros(5), None, "hist").shape == (5,)
    bad = [np.zeros(8, np.float32), np.zeros(16)[::2], np.zeros((2, 4)), np.zeros(7), [0.0] * 8]
    ro = np.zeros(8)
    ro.flags.writeable = False
    bad.append(ro)
    for b in bad:
        with pytest.raises(ValueError):
            _out64(b, 8, "out")
    with pytest.raises(ValueError):
        _out64(np.zeros(4, np.float32), None, "hist")
