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
    """bench.py's N > 1 path (NCCL group, max-over-ranks reductions, the chunked trace / NCCL hit
    gather pipeline of one tile-sharded frame, per-rank e2e) exercised on the one GPU of the box
    (--force-dist)."""
    # launches per step: each trace launch is preceded by the two VF_TRACE_SCHEDULE order kernels
    for gather, launches in (("nccl", 2 * 3 * 3), ("p2p", 3 * 3)):
        r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--force-dist", "--config", "cfg2",
                            "--no-cpu-baseline", "--no-side", "--steps", "3", "--warmup", "3", "--gather-chunks", "2",
                            "--gather", gather], capture_output=True, text=True, timeout=600, cwd=ROOT)
        assert r.returncode == 0, r.stderr[-3000:]
        d = json.loads([l for l in r.stdout.splitlines() if l.strip()][-1])
        assert d["value"] > 0 and d["scaling"] == "strong" and d["gpu_launches"] == launches and d["e2e"]["value"] > 0
        assert d["trace_only"] >= 0.9 * d["value"]
        assert ("peer memory" in d["config"]["parallelism"]) == (gather == "p2p"), d["config"]["parallelism"]
        assert "replicas verified on 1 rank" in d["config"]["parallelism"], d["config"]["parallelism"]


@pytest.mark.gpu
def test_driver_command_prints_one_compact_json_line():
    """The driver's exact command: the last stdout line parses, is under 4 KB and carries the
    headline, roofline, cpu_baseline, e2e and clocks (VERDICT r1 Missing #1)."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "1", "--steps", "20", "--warmup", "5"],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1 and len(lines[0]) < 4096, len(lines[0])
    d = json.loads(lines[0])
    assert d["n_gpus"] == 1 and d["steps"] == 20 and d["warmup"] == 5 and d["value"] > 0
    for k in ("roofline", "cpu_baseline", "e2e", "clocks", "gpu_launches"):
        assert d.get(k), k
    assert d["cpu_baseline"]["parity_mismatches"] == 0 and d["cpu_baseline"]["parity_checked"] > 0
    assert 0 < d["roofline"]["frac"] < 1 and d["e2e"]["h2d_bytes_per_step"] == 32 * d["config"]["rays_per_frame"]
    assert len(d["config"]["rays_sha256"]) == 16  # every ray buffer recorded by its SHA-256


def test_gpus_mismatch_exits_nonzero():
    env = dict(os.environ, RANK="0", WORLD_SIZE="2", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "4", "--steps", "1"],
                       capture_output=True, text=True, timeout=120, cwd=ROOT, env=env)
    assert r.returncode != 0 and "WORLD_SIZE" in r.stderr
