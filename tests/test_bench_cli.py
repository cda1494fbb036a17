"""bench.py's launch contract on CPU: `--gpus N` without a launcher re-executes itself under
torch.distributed.run with N ranks (127.0.0.1 rendezvous); the reference arm (the CPU oracle) runs
on gloo, only rank 0 works and prints exactly one JSON line, whose ms_per_step is what its steps
actually took (a bounded sample of the workload, value scaled to the full grid)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("n", [1, 2])
def test_reference_arm_spawns_ranks(n):
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    env.pop("RANK", None)
    env.pop("LOCAL_RANK", None)
    cmd = [sys.executable, "bench.py", "--impl", "reference", "--gpus", str(n), "--config", "C2",
           "--steps", "2", "--warmup", "1", "--ref-seconds", "0.5"]
    p = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, p.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == n and d["unit"] == "iter/s" and d["value"] > 0
    if n > 1:
        for r in range(n):
            assert f"rank {r}/{n} process group backend gloo" in p.stderr
    # self-consistent: the K steps' own time fits in the run's wall time
    assert d["ms_per_step"] * d["steps"] / 1000.0 <= d["wall_s"]
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["cpu_model"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
