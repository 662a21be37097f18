"""bench.py's multi-rank entry point on CPU: `bench.py --gpus N` run directly (no torchrun)
spawns N ranks itself ("What's missing" 1); the dry run does only the rank plumbing."""
from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("n", [2, 3])
def test_gpus_n_spawns_n_ranks(n):
    env = dict(os.environ, PYRIT_B200_BENCH_DRYRUN="1", PYRIT_B200_DIST_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    env.pop("RANK", None)
    r = subprocess.run([sys.executable, "bench.py", "--gpus", str(n), "--steps", "3", "--warmup", "3"], cwd=ROOT,
                       env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["world_size"] == n and d["comm_nranks"] == n and d["requested_gpus"] == n
    assert d["spawned_by_bench"] is True


def test_gpus_1_runs_in_process():
    env = dict(os.environ, PYRIT_B200_BENCH_DRYRUN="1")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, "bench.py", "--steps", "3", "--warmup", "3"], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][0])
    assert d["world_size"] == 1 and d["spawned_by_bench"] is False


@pytest.mark.gpu
def test_gpus_2_full_bench_on_gpu():
    """The whole N-rank bench path on the GPU box, no torchrun: `bench.py --gpus 2` spawns
    two ranks (sharing the one visible GPU over gloo), each encodes its byte-offset shard of
    config 2, the step time is reduced over ranks, every rank's shard is compared byte for
    byte with the reference's CPU output, and rank 0 alone prints the line."""
    env = dict(os.environ, PYRIT_B200_DIST_BACKEND="gloo", PYRIT_B200_TIERED="0")
    env.pop("WORLD_SIZE", None)
    env.pop("RANK", None)
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--config", "2", "--steps", "5", "--warmup", "3",
                        "--no-cpu-baseline"], cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["ranks"]["ok"] and d["ranks"]["spawned_by_bench"]
    assert d["verified"] is True
    assert d["verification"]["reference"]["identical"] is True
    assert d["value"] > 0 and d["gpu_launches"] > 0
