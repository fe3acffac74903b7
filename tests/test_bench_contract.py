"""bench.py keeps the driver's JSON-line contract.

CPU: the reference arm (the oracle, --impl reference) prints one line with the
required keys.  GPU: our arm prints one line with value / roofline /
cpu_baseline / e2e / gpu_launches / clocks, and the device numbers are
internally consistent.
"""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
             "scaling", "vs_baseline", "dtype", "data", "config"}


def run_bench(*args, timeout=900):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    d = run_bench("--impl", "reference", "--workload", "cfg1", "--steps", "2", "--warmup", "3")
    assert BASE_KEYS <= set(d)
    assert d["impl"] == "reference" and d["value"] > 0 and d["warmup"] >= 3
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["unit"] == d["unit"]


@pytest.mark.gpu
def test_our_arm_line():
    d = run_bench("--workload", "cfg2", "--steps", "5", "--warmup", "3", "--no-cpu-baseline")
    assert BASE_KEYS <= set(d)
    assert d["n_gpus"] == 1 and d["value"] > 0 and d["gpu_launches"] >= 5
    roof = d["roofline"]
    assert roof["bound"] == "alu" and 0 < roof["frac"] < 1 and abs(roof["achieved"] / roof["peak"] - roof["frac"]) < 1e-9
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] == 4096 * 1024 * 8
    assert d["step_ms"]["min"] <= d["step_ms"]["median"] <= d["step_ms"]["p90"]
    assert "sm_mhz" in d["clocks"]
    # the timed outputs equal the oracle's (gathered per-unit digests vs tests/golden)
    assert d["digests_ok"] is True and d["gpus_active"] == 1
    assert d["digests"]["e2e_outputs_equal_device_outputs"] is True
    # value = limb-transforms per step / step time
    assert abs(d["value"] - 2 * 4096 / (d["ms_per_step"] * 1e-3)) / d["value"] < 1e-6
