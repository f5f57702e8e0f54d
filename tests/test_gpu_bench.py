"""bench.py contract on the GPU (small n so it runs in seconds): one JSON line on
stdout with every key the driver reads, sane values, and the CUDA path loaded."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("n", [4096, 8192])
def test_bench_json_contract(n):
    out = subprocess.run([sys.executable, "bench.py", "--size", str(n), "--steps", "5", "--warmup", "3",
                          "--cpu-steps", "1"], cwd=ROOT, capture_output=True,
                         text=True, timeout=600, check=True).stdout
    lines = out.strip().splitlines()
    assert len(lines) == 1, out                      # exactly one JSON line on stdout
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e",
              "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 5 and d["warmup"] == 3 and d["value"] > 0
    assert abs(d["ms_per_step"] * d["value"] - 1e3) < 1e-6 * 1e3
    assert "workload" in d["config"] and "model" not in d["config"]
    rf = d["roofline"]
    assert rf["bound"] == "hbm" and rf["unit"] == "GB/s" and rf["achieved"] > 0 and rf["peak"] > 0
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-12
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] > 0 and cb["sample"]
    assert cb["one_thread"]["cores"] == 1 and cb["one_thread"]["value"] > 0
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == 16 * n and e["d2h_bytes_per_step"] == 16 * (n + 1)
    assert d["gpu_launches"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    if n == 4096:
        assert "small" in rf["kernel"]
