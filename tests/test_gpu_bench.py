"""bench.py's JSON contract on the GPU (the driver parses this line): one line with the metric,
value, roofline (dominant kernel, algorithmic bytes over its CUDA-event time), cpu_baseline (the
oracle), e2e (host buffers through the C ABI, with the bytes copied), clocks and gpu_launches, on a
small config so the test stays short."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_line_contract():
    pytest.importorskip("torch")
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"):
        env.pop(k, None)
    cmd = [sys.executable, "bench.py", "--config", "C3", "--steps", "3", "--warmup", "3", "--no-trisor",
           "--ref-seconds", "1"]
    p = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "clocks",
              "gpu_launches", "time_to_solution"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["value"] > 0
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0.2 < r["frac"] < 1.2
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert d["e2e"]["h2d_bytes_per_step"] == d["e2e"]["d2h_bytes_per_step"] == 8 * 640 * 480 * 70
    assert 0 < d["e2e"]["value"] <= d["value"] * 1.05
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["gpu_launches"] > 0
    # the iterations of the timed steps: 8 per step, nothing skipped
    assert d["config"]["iters_per_step"] == 8
    assert abs(d["value"] - 8 * 3 / (d["ms_per_step"] * 3 / 1000.0)) / d["value"] < 1e-6
