"""Benchmark: batched SPHINCS+ signing throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--set 128f] [--count 4096]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N
    python bench.py --impl reference ...      # the CPU reference arm

Workload (BASELINE.json configs[1]): SPHINCS+-128f, 4096 synthetic 32-byte
messages per GPU, one key, rng = random.Random(2512_23969).
A step signs the whole batch: one CUDA-graph launch of msg_prep ->
{FORS_Sign -> T_k} || TREE_Sign -> WOTS_Sign.  Weak scaling: each rank signs
its own 4096-message shard; no collective is on the signing path (the only
torch.distributed traffic is the barrier and the max-over-ranks of times).

value  : whole-job signatures/s with inputs resident in HBM (device-timed,
         CUDA events per step on the launching stream, L2 flushed between
         steps by rewriting a 256 MiB buffer outside the events).
e2e    : the same metric through the public API (hs_sign_batch via
         Engine.sign_into) from pinned host buffers: H2D of the messages,
         signing, D2H of every signature, each step; host wall clock.
roofline: TREE_Sign (the dominant kernel, ~89% of 128f work) against the
         B200 integer-issue roofline N_SM * f_max * 128 / 1384 compressions/s
         (SURVEY.md s.8(d)); its duration is taken with CUDA events around the
         kernel in a serialised run (hs_run mode 1) inside this process.
cpu_baseline: the C restatement of the reference signer (oracle/, a "port"),
         all host threads, a bounded sample of the same workload.
launch_latency: the metric's "batch launch latency": host time inside the
         one cudaGraphLaunch per batch, device batch time, public-API wall
         time per batch, and small-batch (1 / 64 message) API latency.
other_sets: the same measurements for the other two parameter sets at their
         BASELINE batch sizes (192f: 16384 messages per GPU, configs[2];
         256f: 65536, configs[3] -- signed as 4 chunk launches of 16384 over
         resident inputs), each with its own CPU baseline, so one default run
         covers 128f/192f/256f; --single-set skips them.
--gpus N: one process per GPU.  Under torchrun WORLD_SIZE must equal N;
         launched plainly with N > 1, bench.py spawns the N ranks itself
         (RANK / LOCAL_RANK / WORLD_SIZE, rendezvous on 127.0.0.1) and relays
         rank 0's line; --plan prints that launch plan without running.
"""

from __future__ import annotations

import argparse
import json
import os
import platform
import random
import socket
import ssl
import statistics
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

SEED = 2512_23969
OPS_PER_COMPRESSION = 1384     # canonical integer ops of one SHA-256 compression
ISSUE_PER_CLK_PER_SM = 128     # 4 SMSPs x 32 lanes


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--set", dest="set_id", default="128f", choices=["128f", "192f", "256f"])
    ap.add_argument("--count", type=int, default=4096, help="messages per GPU per step")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="target CPU-baseline sample length")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--check", type=int, default=16, help="signatures checked vs the oracle after timing")
    ap.add_argument("--single-set", action="store_true", help="skip the secondary sets (other_sets)")
    ap.add_argument("--plan", action="store_true", help="print the rank launch plan as JSON and exit")
    return ap.parse_args()


# BASELINE.json configs each set's batch size comes from
BASELINE_CONFIG = {("128f", 4096): "configs[1]", ("192f", 16384): "configs[2]", ("256f", 65536): "configs[3]"}


def bench_config(set_id: str, count: int, gpus: int) -> dict:
    """The workload both arms report (identical dicts, so the driver can match
    the reference arm's line to ours)."""
    return {"workload": f"SPHINCS+-{set_id} batched sign, {count} x 32-byte msgs per GPU, 1 key",
            "set": set_id, "messages_per_gpu": count, "message_bytes": 32, "keys": 1, "global_batch": gpus * count,
            "parallelism": f"message-shard x{gpus}",
            "baseline_config": BASELINE_CONFIG.get((set_id, count), "custom")}


def host_info() -> dict:
    """CPU model and the versions BASELINE.md s.3 asks to report beside a CPU baseline."""
    model = platform.processor() or ""
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu_model": model, "logical_cpus": os.cpu_count(), "python": platform.python_version(),
            "openssl": ssl.OPENSSL_VERSION}


def free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def rank_plan(gpus: int, port: int) -> list[dict]:
    """Environment of each rank when bench.py launches the N processes itself
    (the same variables torchrun sets; one process per GPU, LOCAL_RANK picks it)."""
    return [{"RANK": str(r), "LOCAL_RANK": str(r), "WORLD_SIZE": str(gpus), "LOCAL_WORLD_SIZE": str(gpus),
             "MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port)} for r in range(gpus)]


def spawn_ranks(gpus: int) -> int:
    """Run this script once per GPU and relay rank 0's stdout (its JSON line)."""
    plan = rank_plan(gpus, free_port())
    procs = []
    for env in plan:
        procs.append(subprocess.Popen([sys.executable, str(Path(__file__).resolve())] + sys.argv[1:],
                                      env=dict(os.environ, **env),
                                      stdout=subprocess.PIPE if env["RANK"] == "0" else subprocess.DEVNULL))
    out, _ = procs[0].communicate()
    rc = max(abs(pr.wait()) for pr in procs)
    sys.stdout.write(out.decode())
    sys.stdout.flush()
    return rc


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def rank_device(local: int) -> int:
    """This rank's GPU: LOCAL_RANK.  HS_BENCH_ONE_DEVICE=1 puts every rank on
    device 0 -- a check of the N-rank launch / barrier / max-over-ranks path on
    a one-GPU box (the line then carries "ranks_share_device": true and its
    numbers are not a scaling measurement)."""
    return 0 if os.environ.get("HS_BENCH_ONE_DEVICE") == "1" else local


def init_dist(world: int):
    if world <= 1:
        return None
    import torch.distributed as dist

    dist.init_process_group(backend="gloo")
    return dist


def max_over_ranks(dist, v: float) -> float:
    if dist is None:
        return v
    import torch

    t = torch.tensor([v], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(dist):
    if dist is not None:
        dist.barrier()


def workload(set_id: str, count: int, rank: int):
    """BASELINE.md s.3 recipe; rank r's shard continues the same RNG stream."""
    from paper_2512_23969_b200.params import derive

    p = derive(set_id)
    rng = random.Random(SEED)
    seed = rng.randbytes(3 * p.n)
    for _ in range(rank * count):
        rng.randbytes(32)
    msgs = [rng.randbytes(32) for _ in range(count)]
    return p, seed, msgs


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.out = ""

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        time.sleep(0.15)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                self.out = ""

    def summary(self) -> dict:
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.out.splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                clk, cmax = float(f[1]), float(f[2])
            except ValueError:
                continue
            mx = max(mx, cmax)
            sm.append(clk)
            for name, val in zip(names, f[5:9]):
                if val.lower() in ("active", "1"):
                    reasons.add(name)
        loaded = [c for c in sm if c > 0.5 * mx] if mx else sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_sign_rate(set_id: str, sk: bytes, msgs: list[bytes], seconds: float, threads: int):
    """Oracle port (C, all host threads) on a bounded sample; returns (sig/s, sample size, wall s)."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle  # CPU baseline leg only

    oracle.build()
    probe = msgs[: max(threads, 8)]
    t0 = time.perf_counter()
    oracle.sign_many(set_id, sk, None, probe, threads=threads)
    dt = time.perf_counter() - t0
    rate0 = len(probe) / max(dt, 1e-9)
    n = int(min(len(msgs) * 4, max(threads * 2, rate0 * seconds)))
    sample = [msgs[i % len(msgs)] for i in range(n)]
    t0 = time.perf_counter()
    oracle.sign_many(set_id, sk, None, sample, threads=threads)
    dt = time.perf_counter() - t0
    return n / dt, n, dt


def cpu_baseline_line(set_id: str, sk: bytes, msgs: list[bytes], seconds: float) -> dict:
    """cpu_baseline object: the oracle port on every host thread, a bounded sample."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle  # CPU baseline leg only

    threads = os.cpu_count() or 1
    rate, n, dt = cpu_sign_rate(set_id, sk, msgs, seconds, threads)
    return {"value": round(rate, 3), "unit": "sig/s", "cores": threads, "kind": "port",
            "sample": f"{n} of the same {set_id} messages in {dt:.1f}s, C oracle (oracle/hs_oracle.c, "
                      f"SHA-NI={oracle.shani_active()})", **host_info()}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle  # reference arm: the CPU restatement of the reference signer

    oracle.build()
    p, seed, msgs = workload(args.set_id, args.count, 0)
    sk = oracle.keygen(args.set_id, seed)
    threads = os.cpu_count() or 1
    rate_probe, _, _ = cpu_sign_rate(args.set_id, sk, msgs, 1.0, threads)
    per_step = int(max(threads, min(args.count, rate_probe * max(1.0, 60.0 / max(1, args.steps + args.warmup)))))
    for _ in range(args.warmup):
        oracle.sign_many(args.set_id, sk, None, msgs[:threads], threads=threads)
    times = []
    for s in range(args.steps):
        batch = [msgs[(s * per_step + i) % len(msgs)] for i in range(per_step)]
        t0 = time.perf_counter()
        oracle.sign_many(args.set_id, sk, None, batch, threads=threads)
        times.append(time.perf_counter() - t0)
    value = per_step * len(times) / sum(times)
    line = {
        "impl": "reference", "metric": f"signatures/sec SPHINCS+-{args.set_id}", "value": round(value, 3),
        "unit": "sig/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * statistics.mean(times), 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": bench_config(args.set_id, args.count, args.gpus),
        "cpu_baseline": {"value": round(value, 3), "unit": "sig/s", "cores": threads, "kind": "port",
                         "sample": f"{per_step} of the workload's signatures per step x {args.steps} steps, C "
                                   f"oracle (oracle/hs_oracle.c, SHA-NI={oracle.shani_active()})", **host_info()},
        "e2e": {"value": round(value, 3), "unit": "sig/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def measure_set(eng, info, set_id: str, count: int, steps: int, warmup: int, rank: int, world: int, dist,
                check: int, small_batches=(1, 64)) -> dict:
    """Every number of one bench line for one parameter set (device value, no-sharing value,
    TREE_Sign roofline, e2e through the public API, batch launch latency, parity spot check)."""
    import numpy as np

    import paper_2512_23969_b200 as hs
    from paper_2512_23969_b200.engine import PinnedBuffer, pack_messages

    p, seed, msgs = workload(set_id, count, rank)
    sk = eng.keygen_batch(set_id, [seed])[0]
    eng.upload_keys(set_id, sk)
    blob, offs = pack_messages(msgs)
    cfg = eng.config(set_id)
    chunk = min(count, cfg["chunk"])  # messages per graph launch

    # ---- value: inputs resident in HBM, device-timed graph launches ----
    eng.stage(set_id, blob, offs, count)
    flush = 256 << 20
    eng.bench_run(set_id, count, max(1, warmup), 0, flush)
    shape = eng.batch_info(set_id)
    shared_L = shape["shared_layers"]  # depth the auto policy chose for this batch
    launches0 = eng.launch_count
    eng.launch_stats(reset=True)
    barrier(dist)
    with ClockSampler(eng.device) as clocks:
        step_ms = eng.bench_run(set_id, count, steps, 0, flush)
    launches = eng.launch_count - launches0
    lstat = eng.launch_stats(reset=True)
    barrier(dist)
    dev_s = max_over_ranks(dist, sum(step_ms) / 1e3)
    value = world * count * steps / dev_s
    graph_ms = eng.timings()

    # ---- the same batch with subtree sharing off (every message recomputes every layer) ----
    value_plain = None
    if shared_L:
        eng.set_config(set_id, shared_layers=0)
        eng.stage(set_id, blob, offs, count)
        eng.bench_run(set_id, count, max(1, warmup), 0, flush)
        barrier(dist)
        plain_ms = eng.bench_run(set_id, count, steps, 0, flush)
        plain_s = max_over_ranks(dist, sum(plain_ms) / 1e3)
        value_plain = world * count * steps / plain_s
        eng.set_config(set_id, shared_layers=cfg["shared_layers"])

    # ---- per-kernel roofline (serialised run of one launch's chunk, CUDA events around each kernel) ----
    rblob, roffs = pack_messages(msgs[:chunk])
    eng.stage(set_id, rblob, roffs, chunk)
    eng.bench_run(set_id, chunk, 1, 1, flush)
    kt = [eng.timings()]
    tree_ms = []
    for _ in range(3):
        eng.bench_run(set_id, chunk, 1, 1, flush)
        tree_ms.append(eng.timings()["TREE_Sign"])
    tree_ms_avg = statistics.mean(tree_ms)
    rinfo = eng.batch_info(set_id)
    rshared_L = rinfo["shared_layers"]
    units = rinfo["shared_subtrees_built"]  # shared subtrees the launch actually read
    work = hs.compressions_per_signature(p, 32)
    sub = hs.params.subtree_compressions(p)
    # executed compressions of the timed per-message TREE_Sign kernel (the
    # subtrees below the shared layers); the shared-subtree kernel (`units`
    # subtrees of the single key, run concurrently in the graph) is counted in
    # executed_per_sig but not in the roofline kernel
    tree_comps = chunk * (p.d - rshared_L) * sub
    achieved = tree_comps / (tree_ms_avg / 1e3)
    clk = clocks.summary()
    sm_max = clk.get("sm_max_mhz") or 1965.0
    peak = info["sm_count"] * sm_max * 1e6 * ISSUE_PER_CLK_PER_SM / OPS_PER_COMPRESSION
    traffic = None
    tpath = ROOT / "profiles" / "tree_traffic.json"
    if tpath.exists():
        try:
            traffic = json.loads(tpath.read_text()).get(set_id, {}).get("bytes_per_launch_per_msg")
            traffic = traffic * chunk if traffic is not None else None
        except (ValueError, AttributeError):
            traffic = None
    executed_per_sig = (work["host"] + work["FORS_Sign"] + (tree_comps + units * sub) / chunk
                        + (0 if cfg["wots_from_tree"] else work["WOTS_Sign"]))
    per_gpu = value / world
    step_fracs = {
        "reference_count": round(per_gpu * work["total"] / peak, 4),
        "executed_count": round(per_gpu * executed_per_sig / peak, 4),
        "no_subtree_sharing": round(value_plain / world * work["total"] / peak, 4) if value_plain else None,
        "note": "whole-step compressions/s per GPU / int-issue peak: at the reference's count per signature "
                "(what a signature is worth), at the count the kernels execute (subtree sharing computes the "
                "top layers once per batch), and with sharing off (every message computes every layer)",
    }

    # ---- e2e: public API, pinned host buffers, H2D + sign + D2H every step ----
    h_blob = PinnedBuffer(max(len(blob), 1))
    h_blob.array()[: len(blob)] = np.frombuffer(blob, dtype=np.uint8)
    h_offs = PinnedBuffer(offs.nbytes)
    h_offs.array(np.uint64)[:] = offs
    h_out = PinnedBuffer(count * p.sig_bytes)
    for _ in range(max(1, warmup)):
        eng.sign_into(set_id, h_blob.ptr, h_offs.array(np.uint64), count, h_out.ptr)
    barrier(dist)
    eng.launch_stats(reset=True)
    t0 = time.perf_counter()
    for _ in range(steps):
        eng.sign_into(set_id, h_blob.ptr, h_offs.array(np.uint64), count, h_out.ptr)
    e2e_s = max_over_ranks(dist, time.perf_counter() - t0)
    e2e_launch = eng.launch_stats(reset=True)
    e2e = world * count * steps / e2e_s
    sigs_out = bytes(h_out.view[: count * p.sig_bytes])

    # ---- small-batch latency through the same public call (serving-shaped) ----
    small = {}
    for nb in small_batches:
        nb = min(nb, count)
        for _ in range(3):
            eng.sign_into(set_id, h_blob.ptr, h_offs.array(np.uint64)[: nb + 1], nb, h_out.ptr)
        lat = []
        for _ in range(10):
            t1 = time.perf_counter()
            eng.sign_into(set_id, h_blob.ptr, h_offs.array(np.uint64)[: nb + 1], nb, h_out.ptr)
            lat.append(time.perf_counter() - t1)
        small[str(nb)] = round(1e6 * statistics.median(lat), 1)
    # the same small batches' device time (graph, inputs staged; CUDA events)
    small_dev = {}
    for nb in small_batches:
        nb = min(nb, count)
        eng.stage(set_id, blob[: int(offs[nb])], offs[: nb + 1], nb)
        eng.bench_run(set_id, nb, 3, 0)
        small_dev[str(nb)] = round(1e3 * statistics.median(eng.bench_run(set_id, nb, 10, 0)), 1)
    eng.launch_stats(reset=True)

    # ---- correctness spot check of the timed e2e output vs the oracle ----
    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle  # checker

    oracle.build()
    chk = list(range(0, count, max(1, count // max(1, check))))[:check]
    ref, _ = oracle.sign_many(set_id, sk, None, [msgs[i] for i in chk])
    ok = all(sigs_out[i * p.sig_bytes:(i + 1) * p.sig_bytes] == r for i, r in zip(chk, ref))
    ok_all = max_over_ranks(dist, 0.0 if ok else 1.0) == 0.0
    for b in (h_blob, h_offs, h_out):
        b.free()

    return {
        "p": p, "sk": sk, "msgs": msgs, "cfg": cfg, "clk": clk, "value": value, "dev_s": dev_s,
        "value_plain": value_plain, "launches": launches, "shared_L": shared_L, "units": units,
        "e2e": {"value": round(e2e, 1), "unit": "sig/s", "h2d_bytes_per_step": int(len(blob) + offs.nbytes),
                "d2h_bytes_per_step": int(count * p.sig_bytes)},
        "launch_latency": {
            "graph_launches_per_batch": round(lstat["graph_launches"] / max(1, steps), 3),
            "host_graph_launch_us": {"mean": round(lstat["mean_us"], 2), "max": round(lstat["max_us"], 2)},
            "device_batch_us": round(1e3 * statistics.median(step_ms), 1),
            "e2e_batch_us": round(1e6 * e2e_s / steps, 1),
            "e2e_graph_launches_per_batch": round(e2e_launch["graph_launches"] / max(1, steps), 3),
            "e2e_small_batch_us": small,
            "device_small_batch_us": small_dev,
            "note": "host time inside cudaGraphLaunch (one graph per batch of up to `chunk` messages); device "
                    "batch time (CUDA events); public-API wall time per batch incl. H2D/D2H; median wall time of "
                    "small batches (messages: us) and their device graph time",
        },
        "roofline": {
            "bound": "int-issue",
            "kernel": "TREE_Sign",
            "achieved": round(achieved / 1e9, 3),
            "peak": round(peak / 1e9, 3),
            "unit": "Gcompressions/s",
            "frac": round(achieved / peak, 4),
            "traffic": traffic,
            "traffic_gbs": round(traffic / (tree_ms_avg / 1e3) / 1e9, 1) if traffic else None,
            "traffic_note": "DRAM bytes of the per-message TREE_Sign kernels (profiles/tree_traffic.json, ncu): the "
                            "signing leaf's 16 chain positions per chain kept for the WOTS gather (the digits are "
                            "known only once the layer below is signed) and the chain ends written once and read "
                            "once by the leaf grid -- a few % of HBM bandwidth next to an integer-issue-bound kernel",
            "work_per_launch": f"{chunk} msgs x {p.d - rshared_L} layers x {sub} compressions per subtree "
                               f"(executed; {rshared_L} top layers come from {units} shared subtrees)",
            "kernel_ms": round(tree_ms_avg, 3),
            "peak_basis": f"{info['sm_count']} SMs x {sm_max:.0f} MHz x 128 / 1384",
        },
        "step_fracs": step_fracs,
        # graph mode times the whole batch (and msg_prep); the per-kernel split
        # comes from the serialised run below, so unmeasured zeros are dropped
        "kernel_ms_graph": {k: round(v, 3) for k, v in graph_ms.items() if v > 0},
        "kernel_ms_serial": {k: round(v, 3) for k, v in kt[0].items()},
        "hbm_sig_writeout_gbs": round(count * p.sig_bytes / (statistics.mean(step_ms) / 1e3) / 1e9, 3),
        "compressions_per_sig": {"reference_count": work["total"], "executed": round(executed_per_sig, 1)},
        "parity_spot_check": {"checked": len(chk), "ok": ok_all},
    }


# per-GPU message counts of the sets reported beside the headline (BASELINE
# configs[1..3]: 128f at 4096, 192f at 16384, 256f at 65536 messages)
OTHER_SETS = {"128f": 4096, "192f": 16384, "256f": 65536}


def engine_config(cfg: dict) -> dict:
    return {k: v for k, v in cfg.items() if k.startswith("fors") or k in ("variant", "streams", "chunk",
                                                                        "shared_layers", "tree_split", "overlap")}


def run_ours(args):
    rank, world, local = dist_env()
    dist = init_dist(world)

    import paper_2512_23969_b200 as hs

    eng = hs.get_engine(rank_device(local))
    info = eng.device_info()
    count = args.count
    r = measure_set(eng, info, args.set_id, count, args.steps, args.warmup, rank, world, dist, args.check)
    cpu_ok = rank == 0 and world == 1 and not args.no_cpu_baseline

    others = {}
    if not args.single_set:
        for sid, n in OTHER_SETS.items():
            if sid == args.set_id:
                continue
            o = measure_set(eng, info, sid, n, min(args.steps, 5), args.warmup, rank, world, dist, 4,
                            small_batches=(1,))
            others[sid] = {
                "value": round(o["value"], 1), "unit": "sig/s", "messages_per_gpu": n,
                "config": bench_config(sid, n, world), "engine_config": engine_config(o["cfg"]),
                "ms_per_step": round(1e3 * o["dev_s"] / min(args.steps, 5), 4),
                "value_no_subtree_sharing": round(o["value_plain"], 1) if o["value_plain"] else None,
                "subtree_sharing_layers": o["shared_L"],
                "e2e": o["e2e"], "launch_latency": o["launch_latency"],
                "roofline": {k: o["roofline"][k] for k in ("achieved", "peak", "unit", "frac", "kernel_ms",
                                                           "work_per_launch")},
                "step_fracs": o["step_fracs"],
                "clocks": {"sm_mhz": o["clk"]["sm_mhz"], "reasons": o["clk"]["reasons"]},
                "parity_spot_check": o["parity_spot_check"],
                "cpu_baseline": (cpu_baseline_line(sid, o["sk"], o["msgs"], args.cpu_seconds / 2)
                                 if cpu_ok else None),
            }

    cpu = cpu_baseline_line(args.set_id, r["sk"], r["msgs"], args.cpu_seconds) if cpu_ok else None

    if rank == 0:
        clk = r["clk"]
        cfg = eng.config(args.set_id)
        line = {
            "metric": f"signatures/sec SPHINCS+-{args.set_id}",
            "value": round(r["value"], 1),
            "unit": "sig/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(1e3 * r["dev_s"] / args.steps, 4),
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "u32",
            "data": "synthetic",
            "config": bench_config(args.set_id, count, world),
            "timing": {"l2": "flushed between steps (256 MiB rewrite outside the events)",
                       "value": "CUDA events per step on the launching stream, max over ranks",
                       "e2e": "host wall clock around hs_sign_batch_ex from pinned buffers, max over ranks"},
            "engine_config": engine_config(cfg),
            "e2e": r["e2e"],
            "gpu_launches": int(r["launches"]),
            "launch_latency": r["launch_latency"],
            "value_no_subtree_sharing": round(r["value_plain"], 1) if r["value_plain"] else None,
            "subtree_sharing": {"layers": r["shared_L"], "shared_subtrees_built": r["units"],
                                "policy": "shared_auto: a top layer is shared when its subtrees per key are at most "
                                          "twice the key's messages (max 6 layers; 4 for 256f); only the subtrees "
                                          "some message reads are computed",
                                "note": "top hypertree layers address few subtrees per key; each distinct "
                                        "(key, layer, tree) subtree is computed once per batch (bytes unchanged)"},
            "roofline": r["roofline"],
            "step_fracs": r["step_fracs"],
            "kernel_ms_graph": r["kernel_ms_graph"],
            "kernel_ms_serial": r["kernel_ms_serial"],
            "hbm_sig_writeout_gbs": r["hbm_sig_writeout_gbs"],
            "compressions_per_sig": r["compressions_per_sig"],
            "clocks": {"sm_mhz": clk["sm_mhz"], "sm_max_mhz": clk["sm_max_mhz"], "reasons": clk["reasons"]},
            "parity_spot_check": r["parity_spot_check"],
            "cpu_baseline": cpu,
            "other_sets": others or None,
        }
        if world > 1 and rank_device(1) == 0:
            line["ranks_share_device"] = True
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.gpus < 1:
        sys.exit("bench.py: --gpus must be >= 1")
    if "WORLD_SIZE" in os.environ:
        _, world, _ = dist_env()
        if world != args.gpus:
            sys.exit(f"bench.py: launched with WORLD_SIZE={world} but --gpus {args.gpus}")
        if args.plan:
            print(json.dumps({"launcher": "external", "ranks": world}))
            return
    elif args.gpus > 1 and args.impl == "ours":
        if args.plan:
            print(json.dumps({"launcher": "bench.py", "ranks": rank_plan(args.gpus, 0)}))
            return
        sys.exit(spawn_ranks(args.gpus))
    elif args.plan:
        print(json.dumps({"launcher": "none", "ranks": 1}))
        return
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
