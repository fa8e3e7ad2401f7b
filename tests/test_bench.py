"""bench.py's JSON-line contract (the driver parses it): the GPU leg's keys,
roofline / e2e / clocks / step statistics, and the CPU-only reference arm."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def last_json_line(out: str) -> dict:
    lines = [l for l in out.splitlines() if l.startswith("{")]
    assert lines, out[-2000:]
    return json.loads(lines[-1])


def test_step_stats_and_cpu_model():
    sys.path.insert(0, ROOT)
    import bench
    st = bench.step_stats(np.array([1.0, 2.0, 3.0, 4.0]))
    assert st["mean_ms"] == 2.5 and st["median_ms"] == 2.5 and st["min_ms"] == 1.0 and st["max_ms"] == 4.0
    half = 1.96 * np.std([1, 2, 3, 4], ddof=1) / 2.0
    assert st["ci95_ms"] == [round(2.5 - half, 5), round(2.5 + half, 5)]
    assert isinstance(bench.cpu_model(), str)


def test_reference_arm_line():
    """--impl reference runs the oracle on the host (no GPU) and prints the
    same metric with impl, cpu_baseline and a zero-copy e2e."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    j = last_json_line(r.stdout)
    assert j["impl"] == "reference" and j["unit"] == "TFLOP/s" and j["value"] > 0 and j["higher_is_better"]
    assert j["cpu_baseline"]["kind"] == "oracle" and j["cpu_baseline"]["cores"] >= 1
    assert j["e2e"]["h2d_bytes_per_step"] == 0 and j["e2e"]["value"] == j["value"]


@pytest.mark.gpu
def test_bench_line_contract():
    """A short default run: every key the driver and the judge read."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "5", "--warmup", "3",
                        "--no-cpu-baseline", "--soak", "0.2"], capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    j = last_json_line(r.stdout)
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks", "step_stats"):
        assert k in j, k
    assert j["n_gpus"] == 1 and j["steps"] == 5 and j["warmup"] == 3 and j["value"] > 0
    assert j["config"]["workload"].startswith("batched")
    # headline at the paper's precision (fp32) against measured peaks
    assert j["dtype"] == "f32" and j["roofline"]["peak_measured"] is True
    for p in ("fp32_tc", "tf32", "bf16"):
        sub = j["paths"][p]
        assert sub["dtype"].startswith({"fp32_tc": "f32"}.get(p, p)) and sub["value"] > j["value"]
        assert sub["roofline"]["peak_measured"] is True
        assert 0 < sub["roofline"]["frac"] <= 1.0 and sub["clocks"]["sm_mhz"]
    rf = j["roofline"]
    assert rf["bound"] in ("tensor", "hbm", "alu") and 0 < rf["frac"] <= 1.0
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-3
    e = j["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert j["gpu_launches"] >= j["steps"]
    st = j["step_stats"]
    assert st["ci95_ms"][0] <= st["mean_ms"] <= st["ci95_ms"][1]
    assert abs(st["mean_ms"] - j["ms_per_step"]) < 1e-3
