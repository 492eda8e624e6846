"""bench.py's JSON line (the driver's contract) on the small config c1: every
required key, the roofline and cpu_baseline objects, graph-replay timing, and
the reference arm's line."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_bench_line_c1():
    d = _run("--config", "c1", "--steps", "3", "--warmup", "3")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "clocks", "gpu_launches"):
        assert k in d, k
    assert d["metric"] == "randUTV FP64 GFLOP/s" and d["dtype"] == "f64" and d["n_gpus"] == 1
    assert d["steps"] == 3 and d["warmup"] == 3 and d["value"] > 0 and d["gpu_launches"] > 0
    assert "workload" in d["config"] and "cuda_graph" in d["config"]
    r = d["roofline"]
    assert r["bound"] == "tensor" and 0 < r["frac"] <= 1.0 and r["peak"] > 30 and r["unit"] == "TFLOP/s"
    c = d["cpu_baseline"]
    assert c["kind"] == "oracle" and c["cores"] >= 1 and c["value"] > 0
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == 8 * 512 * 512
    assert "sm_mhz" in d["clocks"]


def test_reference_arm_line_c1():
    d = _run("--impl", "reference", "--config", "c1", "--steps", "1", "--warmup", "0")
    assert d["impl"] == "reference" and d["value"] > 0 and d["cpu_baseline"]["kind"] == "oracle"
    assert d["e2e"]["h2d_bytes_per_step"] == 0
