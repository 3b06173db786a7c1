"""bench.py's JSON line on the GPU (contract keys, whole-cycle steps, the three rooflines), on the small
config 1 so that it runs in seconds."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_line_contract():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "1", "--steps", "2",
                        "--warmup", "3", "--no-cpu-baseline"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"):
        assert key in line, key
    assert line["steps"] == 2 and line["config"]["inner_iterations_timed"] == 2 * line["config"]["restart"]
    assert line["value"] > 0 and line["gpu_launches"] > 0
    assert abs(line["ms_per_step"] * line["steps"] / line["config"]["inner_iterations_timed"] * line["value"] / 1e3
               - 1.0) < 1e-6                      # value = inner iterations / s, step = one cycle
    for key in ("roofline_apply", "roofline_vcycle"):
        assert line[key] is not None and line[key]["frac"] > 0
    rv = line["roofline_vcycle"]
    assert rv["roofline_ms_burst"] <= rv["roofline_ms_sustained"]
    # frac = directly timed whole V-cycles; the per-class sums of the profiled solve and the in-solve bound stay
    for key in ("frac_profiled", "measured_ms_per_vcycle", "roofline_ms_per_vcycle_burst", "in_solve"):
        assert key in rv, key
    assert abs(rv["frac"] * rv["measured_ms_per_vcycle"] / rv["roofline_ms_per_vcycle_burst"] - 1.0) < 1e-9
    assert rv["in_solve"]["ms_per_vcycle_upper_bound"] > 0
    assert "input" in line["ops"]
    assert line["e2e"]["h2d_bytes_per_step"] > 0 and line["e2e"]["d2h_bytes_per_step"] > 0
