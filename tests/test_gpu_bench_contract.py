"""GPU: bench.py's JSON line keeps the driver's contract -- one line on
stdout with the metric, the timing keys, e2e with its copy bytes, the
launch count, the roofline of the dominant kernel, clocks, and the
cross-checks (C3 golden PCG counts, e2e counts = device counts)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_line_contract():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "2", "--warmup", "3",
                          "--no-cpu", "--no-design"], capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    b = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "e2e", "gpu_launches", "roofline",
                "cpu_baseline", "clocks"):
        assert key in b, key
    assert b["n_gpus"] == 1 and b["steps"] == 2 and b["warmup"] == 3 and b["higher_is_better"] is True
    assert b["value"] > 0 and b["ms_per_step"] > 0 and b["unit"] == "cell-steps/s"
    assert b["config"]["workload"].startswith("C3 block city 256x256x64")
    e = b["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert e["same_iterations_as_device_leg"] is True
    assert b["gpu_launches"] > 0
    r = b["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 1
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert b["clocks"]["samples"] > 0
    assert b["golden_check"]["pcg_iterations_equal"] is True
