"""world_size-2 gloo checks of the message-sharded (weak-scaling) bench path on CPU.

Each rank signs its own contiguous shard of one synthetic message stream; the
only cross-rank traffic is the barrier and the max-over-ranks of the timings.
"""

from __future__ import annotations

import os
import socket
import subprocess
import sys

import pytest
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank: int, world: int, port: int, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    sys.path.insert(0, str(ROOT))
    import bench

    dist = bench.init_dist(world)
    p, seed, msgs = bench.workload("128f", 8, rank)
    t = bench.max_over_ranks(dist, float(rank + 1))
    bench.barrier(dist)
    q.put((rank, seed, msgs, t))
    dist.destroy_process_group()


def test_sharded_workload_and_max_over_ranks():
    sys.path.insert(0, str(ROOT))
    import bench

    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    out = sorted(q.get(timeout=120) for _ in range(2))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    (_, seed0, m0, t0), (_, seed1, m1, t1) = out
    assert seed0 == seed1                       # one key, replicated
    assert t0 == t1 == 2.0                      # max over ranks
    _, _, both = bench.workload("128f", 16, 0)  # rank shards = consecutive slices of one stream
    assert m0 + m1 == both and not set(m0) & set(m1)


def test_reference_arm_nonzero_ranks_exit_quietly():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "1", "--warmup", "0"],
                       env=env, capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and r.stdout.strip() == ""
