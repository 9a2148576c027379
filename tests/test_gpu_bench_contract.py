"""bench.py keeps the driver's JSON contract: one line from rank 0 with the required keys and types,
the roofline / cpu_baseline / e2e / clocks / gpu_launches objects, and the reference arm's line."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(*args):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, capture_output=True,
                         text=True, timeout=900, check=True).stdout.strip().splitlines()
    lines = [ln for ln in out if ln.startswith("{")]
    assert len(lines) == 1, out
    return json.loads(lines[0])


def test_bench_line_contract():
    j = run_bench("--config", "c1", "--steps", "3", "--warmup", "3", "--e2e-steps", "3")
    for key, typ in [("metric", str), ("value", float), ("unit", str), ("n_gpus", int), ("steps", int),
                     ("warmup", int), ("ms_per_step", float), ("higher_is_better", bool), ("scaling", str),
                     ("dtype", str), ("data", str), ("config", dict), ("gpu_launches", int)]:
        assert isinstance(j[key], typ), key
    assert "vs_baseline" in j and j["n_gpus"] == 1 and j["steps"] == 3 and j["warmup"] >= 3
    assert j["value"] > 0 and j["gpu_launches"] > 0 and "workload" in j["config"]
    r = j["roofline"]
    assert r["bound"] in ("hbm", "tensor") and r["unit"] in ("GB/s", "TFLOP/s")
    assert 0 < r["frac"] <= 1.0 and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    e = j["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    cb = j["cpu_baseline"]
    assert cb["value"] > 0 and cb["cores"] >= 1 and cb["kind"] in ("port", "reference") and cb["sample"]
    clk = j["clocks"]
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(clk)
    assert j["step_ms"]["best"] <= j["step_ms"]["median"] <= j["step_ms"]["worst"]


def test_reference_arm_line():
    j = run_bench("--impl", "reference", "--config", "c1", "--steps", "1", "--warmup", "1")
    assert j["impl"] == "reference" and j["value"] > 0 and j["unit"] == "frames/s"
    assert j["e2e"]["h2d_bytes_per_step"] == 0 and j["cpu_baseline"]["kind"] in ("port", "reference")
