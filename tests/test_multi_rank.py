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
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--gpus", "2", "--steps", "1",
                        "--warmup", "0"],
                       env=env, capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and r.stdout.strip() == ""


def test_bench_plans_ranks():
    """`bench.py --gpus N` without torchrun launches N ranks itself (one per GPU,
    LOCAL_RANK = rank, rendezvous on 127.0.0.1); under a launcher WORLD_SIZE
    must match --gpus."""
    import json

    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--plan"], capture_output=True,
                       text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    plan = json.loads(r.stdout)
    assert plan["launcher"] == "bench.py"
    assert [(x["RANK"], x["LOCAL_RANK"], x["WORLD_SIZE"]) for x in plan["ranks"]] == [("0", "0", "2"), ("1", "1", "2")]
    assert all(x["MASTER_ADDR"] == "127.0.0.1" for x in plan["ranks"])
    env = dict(os.environ, RANK="0", WORLD_SIZE="2", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "4", "--plan"], env=env,
                       capture_output=True, text=True, timeout=120)
    assert r.returncode != 0 and "WORLD_SIZE=2" in r.stderr


def test_bench_arms_report_the_same_config():
    sys.path.insert(0, str(ROOT))
    import bench

    a = bench.bench_config("256f", 65536, 8)
    assert a == bench.bench_config("256f", 65536, 8) and a["baseline_config"] == "configs[3]"
    assert a["global_batch"] == 8 * 65536


def _sign_worker(rank: int, world: int, port: int, q):
    """One rank of the weak-scaling job: sign this rank's shard of the bench
    workload (oracle-backed handle stand-in; no GPU here) and gather the shards
    on rank 0 over gloo."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    sys.path.insert(0, str(ROOT / "oracle"))
    import bench
    import oracle
    from oracle_engine import OracleEngine

    oracle.build()
    dist = bench.init_dist(world)
    p, seed, msgs = bench.workload("128f", 3, rank)
    sk = oracle.keygen("128f", seed)
    eng = OracleEngine(oracle)
    eng.upload_keys("128f", sk)
    sigs = eng.sign_batch("128f", msgs)
    gathered = [None] * world
    dist.all_gather_object(gathered, (rank, msgs, sigs))
    if rank == 0:
        q.put(gathered)
    dist.destroy_process_group()


def test_sharded_signing_gathers_to_single_process_result():
    """Shards signed independently by 2 gloo ranks and gathered equal one process
    signing the concatenated workload (the message split needs no exchange)."""
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "oracle"))
    import bench
    import oracle

    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_sign_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    gathered = q.get(timeout=180)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    msgs = [m for _, ms, _ in sorted(gathered) for m in ms]
    sigs = [s for _, _, ss in sorted(gathered) for s in ss]
    p, seed, both = bench.workload("128f", 6, 0)
    assert msgs == both
    oracle.build()
    sk = oracle.keygen("128f", seed)
    assert sigs == [oracle.sign("128f", sk, m) for m in both]


def test_multi_engine_shards_on_cpu():
    """MultiEngine's shard split and pointer offsets (engine.py) with oracle-backed
    handle stand-ins: 3 handles, 7 ragged messages, mixed keys and opt_rand, into
    one output buffer and one step-count array."""
    import random

    import numpy as np

    sys.path.insert(0, str(ROOT / "tests"))
    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle
    from oracle_engine import OracleHandle, oracle_wots_steps

    from paper_2512_23969_b200.engine import MultiEngine, pack_messages, shard_ranges
    from paper_2512_23969_b200.params import derive

    oracle.build()
    p = derive("128f")
    rng = random.Random(5)
    sks = [oracle.keygen("128f", rng.randbytes(48)) for _ in range(2)]
    msgs = [rng.randbytes(rng.choice([0, 5, 32, 70])) for _ in range(7)]
    kidx = np.array([rng.randrange(2) for _ in msgs], dtype=np.uint32)
    orand = b"".join(rng.randbytes(p.n) for _ in msgs)
    handles = [OracleHandle(oracle, d) for d in (0, 1, 2)]
    multi = MultiEngine([0, 1, 2], engines=handles)
    multi.upload_keys("128f", sks)
    blob, offs = pack_messages(msgs)
    out = bytearray(len(msgs) * p.sig_bytes)
    steps = np.zeros(len(msgs), dtype=np.uint32)
    multi.sign_into("128f", blob, offs, len(msgs), out, kidx, orand, steps)
    assert [h.shards[0][0] for h in handles] == [n for _, n in shard_ranges(len(msgs), 3)] == [3, 2, 2]
    for i, m in enumerate(msgs):
        o = orand[i * p.n:(i + 1) * p.n]
        assert out[i * p.sig_bytes:(i + 1) * p.sig_bytes] == oracle.sign("128f", sks[kidx[i]], m, o)
        assert steps[i] == oracle_wots_steps(oracle, "128f", sks[kidx[i]], m, o)
