"""Host-side logic of bench.py (no GPU): clock-record rules and the reference arm."""
import json
import os
import subprocess
import sys

import bench

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_clock_rules():
    ok = {"sm_mhz": 1900.0, "sm_max_mhz": 1965.0, "reasons": ["sw_power_cap"]}
    assert not bench.clocks_bad(ok)
    assert bench.clocks_bad({"sm_mhz": 1900.0, "sm_max_mhz": 1965.0, "reasons": ["hw_slowdown"]})
    assert bench.clocks_bad({"sm_mhz": 600.0, "sm_max_mhz": 1965.0, "reasons": []})   # leftover lock
    cs = bench.ClockSampler(0)
    cs.lines = ["0, 1965, 1965, 900.1, 0x4, Not Active, Not Active, Not Active, Active",
                "0, 1800, 1965, 950.0, 0x4, Not Active, Not Active, Not Active, Active"]
    s = cs.summary()
    assert s["sm_mhz"] == 1882.5 and s["reasons"] == ["sw_power_cap"] and s["samples"] == 2


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--size", "4096",
                          "--steps", "3", "--warmup", "3"], cwd=ROOT,
                         capture_output=True, text=True, timeout=300, check=True).stdout
    line = json.loads(out.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "oracle"
    assert line["unit"] == bench.UNIT and line["metric"] == bench.METRIC
