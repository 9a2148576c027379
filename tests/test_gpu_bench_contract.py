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


@pytest.fixture(scope="module")
def gpu_line():
    return run_bench("--config", "c1", "--steps", "3", "--warmup", "3", "--e2e-steps", "3")


def test_bench_line_contract(gpu_line):
    j = gpu_line
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
    fr = j["frame_roofline"]
    assert 0 < fr["frac"] <= 1.0 and abs(fr["achieved_gbs"] - fr["algorithmic_bytes_per_frame"] /
                                         (j["ms_per_step"] / 1000.0) / 1e9) < 1e-6 * fr["achieved_gbs"]
    ks = j["k_sweep"]
    assert set(ks["k"]) >= {"1", "4", "8", "16"} and all(v["frames_per_s"] > 0 for v in ks["k"].values())
    assert {"K=1", "K=3", "K=10", "full_blend"} <= set(ks["feature_pass_ms"])
    grid = j["fslam_bench_grid"]
    assert len(grid["rows"]) == 2 * 6 and grid["spec_acceptance_4"] is not None


def test_reference_arm_line(gpu_line):
    j = run_bench("--impl", "reference", "--config", "c1", "--steps", "2", "--warmup", "3")
    assert j["impl"] == "reference" and j["value"] > 0 and j["unit"] == "frames/s"
    assert j["e2e"]["h2d_bytes_per_step"] == 0 and j["cpu_baseline"]["kind"] in ("port", "reference")
    # honest about what ran: one warm-up frame, then the frames actually timed; same config object
    assert j["warmup"] == 1 and 1 <= j["steps"] <= 2 and j["steps_requested"] == 2
    assert j["config"] == gpu_line["config"] and j["metric"] == gpu_line["metric"]


@pytest.mark.parametrize("extra", [[], ["--geo-split"], ["--gather", "nccl"]])
def test_multi_gpu_code_path_one_rank(extra):
    """The N > 1 path (process group, tk_comm over NCCL, D-sharded frame with the fused or NCCL
    all-gather, optional geometry split, the keyframe-parallel block) run as a one-rank group:
    the only multi-GPU coverage a one-GPU box allows; the contract keys must be there."""
    j = run_bench("--config", "c1", "--steps", "3", "--warmup", "3", "--no-e2e", "--no-cpu", "--force-multi",
                  *extra)
    assert j["value"] > 0 and j["multi_gpu"]["ranks"] == 1 and j["keyframe_parallel"]["value"] > 0
    assert "feature-dim shard" in j["config"]["parallelism"]
    assert (j["gather_path"] or "").startswith("p2p" if "--gather" not in extra else "nccl")
    assert j["mapping"]["value"] > 0
