"""bench.py's multi-rank launch (driver contract: `python bench.py --gpus N` must run N ranks).

`--dry-run` runs the same self-launch (torch.distributed.run, 127.0.0.1 rendezvous), rank /
barrier / max-over-ranks / aggregation path on CPU with gloo; only the device time is a
host-side stand-in.  The GPU arm shares every line of that plumbing (bench.py main)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env_extra=None):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR",
                                                             "MASTER_PORT")}
    env.update(env_extra or {})
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=240, env=env, cwd=ROOT)
    return r


def _json_lines(out):
    return [json.loads(l) for l in out.splitlines() if l.startswith("{")]


@pytest.mark.timeout(300)
def test_gpus2_spawns_two_ranks():
    r = _run(["--gpus", "2", "--dry-run", "--steps", "2", "--warmup", "3"])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _json_lines(r.stdout)
    assert len(lines) == 1, r.stdout            # rank 0 alone prints
    d = lines[0]
    assert d["n_gpus"] == 2 and d["ranks"] == [0, 1]
    assert d["config"]["workload"].startswith("c4")
    assert d["config"]["parallelism"] == "ensemble x2 (no collective)"


@pytest.mark.timeout(120)
def test_single_rank_default():
    r = _run(["--dry-run", "--steps", "1"])
    assert r.returncode == 0, r.stderr[-2000:]
    d = _json_lines(r.stdout)[0]
    assert d["n_gpus"] == 1 and d["ranks"] == [0]


@pytest.mark.timeout(120)
def test_world_mismatch_fails_loudly():
    # under a (simulated) torchrun environment of 2 ranks, --gpus 4 must not silently time 2
    r = _run(["--gpus", "4", "--dry-run"], {"WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode == 2 and "WORLD_SIZE" in r.stderr
