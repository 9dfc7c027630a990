"""bench.py's launcher contract (CPU): `--gpus N` outside torchrun spawns N
ranks (one per GPU) with RANK / WORLD_SIZE / LOCAL_RANK set; under torchrun it
runs as the rank it is; `--impl reference --gpus N` stays a single process."""

import json
import re
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def _lines(cmd, env=None):
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=240, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    # (ranks share one stdout: two records may land on one line)
    return [json.loads(m) for m in re.findall(r"\{[^{}]*\}", out.stdout) if "launch_check" in m]


@pytest.mark.timeout(300)
def test_gpus_n_spawns_n_ranks():
    recs = _lines([sys.executable, "bench.py", "--gpus", "3", "--launch-check"])
    assert sorted(r["rank"] for r in recs) == [0, 1, 2]
    assert all(r["world"] == 3 and r["gpus"] == 3 and r["local_rank"] == r["rank"] for r in recs)


def test_gpus_1_runs_in_process():
    recs = _lines([sys.executable, "bench.py", "--launch-check"])
    assert recs == [{"launch_check": True, "rank": 0, "world": 1, "local_rank": 0, "gpus": 1}]


@pytest.mark.timeout(300)
def test_under_torchrun_no_second_spawn():
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    recs = _lines([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                   "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--gpus", "2",
                   "--launch-check"])
    assert sorted(r["rank"] for r in recs) == [0, 1] and all(r["world"] == 2 for r in recs)


def test_reference_arm_is_single_process():
    recs = _lines([sys.executable, "bench.py", "--impl", "reference", "--gpus", "4", "--launch-check"])
    assert len(recs) == 1 and recs[0]["world"] == 1 and recs[0]["gpus"] == 4
