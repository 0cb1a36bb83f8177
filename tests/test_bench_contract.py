"""bench.py's driver contract: the JSON line's keys and their meaning. The reference arm
(the CPU oracle) runs here on CPU; the B200 arm runs under -m gpu on a small C2 prefix."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"}


def _bench(*args, env=None, timeout=600):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT, env={**os.environ, **(env or {})})
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    lines = [x for x in r.stdout.splitlines() if x.startswith("{")]
    return [json.loads(x) for x in lines]


def test_reference_arm_line():
    (line,) = _bench("--impl", "reference", "--steps", "2", "--warmup", "1", "--ref-frames-per-step", "8")
    assert BASE <= set(line) and line["impl"] == "reference"
    assert line["metric"].startswith("sampled frames/sec") and line["unit"] == "frames/s"
    assert line["value"] > 0 and line["higher_is_better"] is True
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] >= 1
    assert line["cpu_baseline"]["value"] == line["value"]
    assert line["e2e"] == {"value": line["value"], "unit": line["unit"], "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}
    assert line["config"]["workload"].startswith("C2")


def test_reference_arm_nonzero_rank_is_silent():
    assert _bench("--impl", "reference", "--steps", "1", "--warmup", "1", env={"RANK": "1", "WORLD_SIZE": "2"}) == []


@pytest.mark.gpu
def test_b200_arm_line():
    (line,) = _bench("--steps", "3", "--warmup", "3", "--frames", "256", "--e2e-frames", "64", "--cpu-seconds", "1")
    assert BASE | {"roofline", "gpu_launches", "clocks", "breakdown"} <= set(line)
    assert line["n_gpus"] == 1 and line["steps"] == 3 and line["warmup"] == 3 and line["scaling"] == "strong"
    assert line["dtype"] == "u8" and line["data"] == "synthetic" and line["vs_baseline"] is None
    assert line["config"]["frames"] == 256 and line["config"]["step_launch"] == "cuda_graph_replay"
    r = line["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and r["achieved"] > 0 and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    e = line["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == 64 * 1920 * 1080 * 3 and e["d2h_bytes_per_step"] > 0
    assert line["gpu_launches"] == 2 * 3  # histogram + shot-diff per step
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(line["clocks"])
    assert line["cpu_baseline"]["kind"] == "oracle"
    assert abs(line["value"] - 256 / (line["ms_per_step"] / 1e3)) < 1e-6 * line["value"]
