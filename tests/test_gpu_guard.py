"""Out-of-bounds writes (compute-sanitizer is not available on the GPU pool): every
solver path and kernel mode runs with 4 KiB canary zones around every library
buffer (KS_GUARD=1, tools/guard_run.py); no zone may be corrupted."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_no_out_of_bounds_writes():
    env = dict(os.environ, KS_GUARD="1")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "guard_run.py")], cwd=ROOT, env=env,
                         capture_output=True, text=True, timeout=1200)
    assert out.returncode == 0, out.stderr[-2000:]
    assert "VIOLATION" not in out.stdout, out.stdout
    assert out.stdout.strip().splitlines()[-1] == "violations 0", out.stdout


def test_guards_off_by_default():
    import paper_1511_07174_b200 as ks
    if "KS_GUARD" in os.environ:
        pytest.skip("KS_GUARD set in this environment")
    with ks.Context(64) as ctx:
        assert ctx.check_guards() == -1


def test_guard_detector_self_test():
    """The detector sees a corrupted zone: KS_GUARD_SELFTEST=1 writes one byte past
    the end of every library buffer at allocation."""
    code = ("import paper_1511_07174_b200 as ks\n"
            "with ks.Context(256) as c:\n"
            "    print('violations', c.check_guards())\n")
    env = dict(os.environ, KS_GUARD="1", KS_GUARD_SELFTEST="1")
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True, text=True,
                         timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    assert int(out.stdout.strip().split()[-1]) > 0, out.stdout
