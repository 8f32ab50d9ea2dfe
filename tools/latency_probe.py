"""Small-batch latency breakdown: device time of the batch graph (CUDA events,
inputs staged) next to the public call's wall time (pinned host buffers,
staging + H2D + graph + D2H), per set and batch size.

    python tools/latency_probe.py [--sets 128f,192f,256f] [--counts 1,4,16,64,256] [--reps 30]
"""

from __future__ import annotations

import argparse
import json
import random
import statistics
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import paper_2512_23969_b200 as hs  # noqa: E402
from paper_2512_23969_b200.engine import PinnedBuffer, pack_messages  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sets", default="128f,192f,256f")
    ap.add_argument("--counts", default="1,4,16,64,256")
    ap.add_argument("--reps", type=int, default=30)
    a = ap.parse_args()
    eng = hs.get_engine(0)
    for set_id in a.sets.split(","):
        p = hs.derive(set_id)
        rng = random.Random(2512_23969)
        sk = eng.keygen_batch(set_id, [rng.randbytes(3 * p.n)])[0]
        eng.upload_keys(set_id, sk)
        for count in [int(c) for c in a.counts.split(",")]:
            msgs = [rng.randbytes(32) for _ in range(count)]
            blob, offs = pack_messages(msgs)
            h_blob = PinnedBuffer(len(blob))
            h_blob.array()[:] = np.frombuffer(blob, dtype=np.uint8)
            h_out = PinnedBuffer(count * p.sig_bytes)
            eng.stage(set_id, blob, offs, count)
            dev = eng.bench_run(set_id, count, a.reps, mode=0)
            for _ in range(5):
                eng.sign_into(set_id, h_blob.ptr, offs, count, h_out.ptr)
            wall = []
            eng.launch_stats(reset=True)
            for _ in range(a.reps):
                t0 = time.perf_counter()
                eng.sign_into(set_id, h_blob.ptr, offs, count, h_out.ptr)
                wall.append(time.perf_counter() - t0)
            gl = eng.launch_stats(reset=True)
            # the same C call without the Python wrapper's argument handling
            from paper_2512_23969_b200 import _lib
            from paper_2512_23969_b200.engine import SET_INDEX
            L = _lib.lib()
            o64 = np.ascontiguousarray(offs, dtype=np.uint64)
            op, bp, sp = o64.ctypes.data, h_blob.ptr, h_out.ptr
            raw = []
            for _ in range(a.reps):
                t0 = time.perf_counter()
                rc = L.hs_sign_batch_ex(eng._h, SET_INDEX[set_id], bp, op, None, None, count, sp, None)
                raw.append(time.perf_counter() - t0)
                assert rc == 0
            info = eng.batch_info(set_id)
            print(json.dumps({"set": set_id, "count": count,
                              "device_graph_us": round(1e3 * statistics.median(dev), 1),
                              "api_wall_us": round(1e6 * statistics.median(wall), 1),
                              "api_wall_min_us": round(1e6 * min(wall), 1),
                              "c_call_us": round(1e6 * statistics.median(raw), 1),
                              "host_graph_launch_us": round(gl["mean_us"], 1),
                              "batch": info}), flush=True)
            h_blob.free()
            h_out.free()


if __name__ == "__main__":
    main()
