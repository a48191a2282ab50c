"""bench.py contract on CPU: the reference arm (this tier's reference = the oracle, as it stands)
prints one JSON line with the keys the driver reads; no GPU needed for this leg."""
from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "cfg1",
                        "--steps", "2", "--warmup", "3"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "config",
              "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["steps"] == 2 and d["warmup"] == 3 and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


def test_reference_arm_nonzero_rank_is_silent():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "cfg1",
                        "--steps", "1", "--warmup", "3"], capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert r.returncode == 0 and r.stdout.strip() == ""


@pytest.mark.gpu
def test_multi_rank_code_path_with_one_rank():
    """bench.py's N > 1 path (NCCL group, max-over-ranks reductions, the strong_frame pipeline of
    chunked traces and NCCL hit gathers, per-rank e2e) exercised on the one GPU of the box
    (--force-dist)."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--force-dist", "--config", "cfg2",
                        "--no-sweep", "--no-cpu-baseline", "--steps", "3", "--warmup", "3", "--gather-chunks", "2"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads([l for l in r.stdout.splitlines() if l.strip()][-1])
    assert d["value"] > 0 and d["scaling"] == "weak" and d["gpu_launches"] == 3 and d["e2e"]["value"] > 0
    sf = d["strong_frame"]  # one frame split over the ranks + NCCL hit gather (north_star)
    assert sf["value"] > 0 and sf["trace_only"] >= 0.9 * sf["value"] and sf["gather_chunks"] == 2
