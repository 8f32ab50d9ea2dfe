"""A/B device timing of one batch under alternative engine configs (same box,
interleaved): python tools/ab_config.py --set 192f --count 16384 \
    --a '{"shared_layers": 4}' --b '{"shared_layers": 5}'"""

from __future__ import annotations

import argparse
import json
import random
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import paper_2512_23969_b200 as hs  # noqa: E402
from paper_2512_23969_b200.tuner import _synthetic  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--set", dest="set_id", default="192f")
    ap.add_argument("--count", type=int, default=16384)
    ap.add_argument("--a", default="{}")
    ap.add_argument("--b", default="{}")
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--serial", action="store_true", help="also time the serialised kernels (one chunk)")
    ap.add_argument("--e2e", action="store_true", help="also time the public call from pinned host buffers")
    a = ap.parse_args()
    eng = hs.get_engine(0)
    base = eng.config(a.set_id)
    cfgs = {"A": json.loads(a.a), "B": json.loads(a.b)}
    res = {"A": [], "B": []}
    info = {}
    ser = {}
    e2e = {}
    pins = {}
    for _ in range(a.rounds):
        for k, c in cfgs.items():
            eng.set_config(a.set_id, **{**base, **c})
            _synthetic(eng, a.set_id, a.count)
            eng.bench_run(a.set_id, a.count, 2, 0, 256 << 20)
            res[k] += eng.bench_run(a.set_id, a.count, a.steps, 0, 256 << 20)
            info[k] = eng.batch_info(a.set_id)
            if a.e2e:  # public call, pinned host buffers, H2D + sign + D2H
                import time

                import numpy as np

                from paper_2512_23969_b200.engine import PinnedBuffer, pack_messages
                from paper_2512_23969_b200.params import derive

                if k not in pins:
                    rng = random.Random(2512_23969)
                    blob, offs = pack_messages([rng.randbytes(32) for _ in range(a.count)])
                    hb = PinnedBuffer(len(blob))
                    hb.array()[: len(blob)] = np.frombuffer(blob, dtype=np.uint8)
                    pins[k] = (hb, offs, PinnedBuffer(a.count * derive(a.set_id).sig_bytes))
                hb, offs, out = pins[k]
                eng.sign_into(a.set_id, hb.ptr, offs, a.count, out.ptr)
                for _ in range(a.steps):
                    t0 = time.perf_counter()
                    eng.sign_into(a.set_id, hb.ptr, offs, a.count, out.ptr)
                    e2e.setdefault(k, []).append(1e3 * (time.perf_counter() - t0))
            if a.serial and a.count <= eng.config(a.set_id)["chunk"]:  # per-kernel times, serialised
                for _ in range(2):
                    eng.bench_run(a.set_id, a.count, 1, 1, 256 << 20)
                    for kn, v in eng.timings().items():
                        ser.setdefault(k, {}).setdefault(kn, []).append(v)
    for k in res:
        ms = statistics.median(res[k])
        print(json.dumps({"cfg": k, "overrides": cfgs[k], "batch": info[k], "median_ms": round(ms, 3),
                          "sig_per_s": round(a.count / ms * 1e3, 1), "all_ms": [round(x, 2) for x in res[k]],
                          "serial_ms": {kn: round(statistics.median(v), 3) for kn, v in ser.get(k, {}).items()},
                          "e2e_median_ms": round(statistics.median(e2e[k]), 3) if k in e2e else None}))


if __name__ == "__main__":
    main()
