"""The driver's multi-GPU bench commands, run end to end on a one-GPU box.

`bench.py --gpus 2` launched plainly (it spawns its two ranks) and under
`torch.distributed.run` (the driver's N>1 command) with HS_BENCH_ONE_DEVICE=1,
which puts both ranks on device 0: the rank launch, the gloo barriers, the
max-over-ranks timing and the single JSON line from rank 0 are exercised with
real signing on each rank (BASELINE configs[3] is multi-GPU; the scaling
numbers themselves need an 8-GPU box).
"""

from __future__ import annotations

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent
ARGS = ["--gpus", "2", "--steps", "3", "--warmup", "3", "--count", "512", "--single-set", "--no-cpu-baseline",
        "--check", "4"]


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(cmd: list[str]) -> dict:
    env = dict(os.environ, HS_BENCH_ONE_DEVICE="1")
    for k in ("RANK", "LOCAL_RANK", "WORLD_SIZE", "LOCAL_WORLD_SIZE", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    p = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout[-2000:]  # one line, from rank 0 only
    return json.loads(lines[0])


def _check(line: dict):
    assert line["n_gpus"] == 2 and line["ranks_share_device"] is True
    assert line["config"]["global_batch"] == 2 * 512
    assert line["value"] > 0 and line["e2e"]["value"] > 0
    assert line["parity_spot_check"]["ok"] is True
    assert line["gpu_launches"] > 0


def test_bench_spawns_its_ranks():
    _check(_run([sys.executable, "bench.py"] + ARGS))


def test_bench_under_torchrun():
    _check(_run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                 "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py"] + ARGS))
