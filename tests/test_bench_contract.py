"""bench.py's JSON line (the driver's contract): the reference arm on the CPU
(small sample) and the GPU arm at a reduced R-MAT scale carry every key the
driver reads, with sane values."""
import json
import os
import subprocess
import sys

import pytest

import oracles

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE = ["metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "e2e", "cpu_baseline"]


def _line(args, timeout):
    p = subprocess.run([sys.executable, "bench.py"] + args, cwd=ROOT, capture_output=True, text=True, timeout=timeout)
    assert p.returncode == 0, p.stderr[-2000:]
    return json.loads(p.stdout.strip().splitlines()[-1])


@pytest.mark.skipif(not oracles.available("ref"), reason="oracle/_ref not built")
@pytest.mark.timeout(600)
def test_reference_arm_line():
    d = _line(["--impl", "reference", "--steps", "1", "--warmup", "0", "--scale", "12", "--cpu-scale", "10"], 600)
    for k in BASE + ["impl"]:
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["config"]["workload"].startswith("config 4")


@pytest.mark.gpu
@pytest.mark.timeout(900)
def test_gpu_arm_line():
    d = _line(["--steps", "2", "--warmup", "1", "--scale", "14", "--cpu-scale", "10"], 900)
    for k in BASE + ["roofline", "gpu_launches", "clocks", "like_for_like"]:
        assert k in d, k
    assert d["value"] > 0 and d["gpu_launches"] > 0 and d["dtype"] == "f64"
    r = d["roofline"]
    assert r["bound"] == "hbm" and 0 < r["frac"] < 1 and r["achieved"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["like_for_like"]["same_rotation_count"] is True
