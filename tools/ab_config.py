"""A/B device timing of one batch under alternative engine configs (same box,
interleaved): python tools/ab_config.py --set 192f --count 16384 \
    --a '{"shared_layers": 4}' --b '{"shared_layers": 5}'"""

from __future__ import annotations

import argparse
import json
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
    a = ap.parse_args()
    eng = hs.get_engine(0)
    base = eng.config(a.set_id)
    cfgs = {"A": json.loads(a.a), "B": json.loads(a.b)}
    res = {"A": [], "B": []}
    info = {}
    for _ in range(a.rounds):
        for k, c in cfgs.items():
            eng.set_config(a.set_id, **{**base, **c})
            _synthetic(eng, a.set_id, a.count)
            eng.bench_run(a.set_id, a.count, 2, 0, 256 << 20)
            res[k] += eng.bench_run(a.set_id, a.count, a.steps, 0, 256 << 20)
            info[k] = eng.batch_info(a.set_id)
    for k in res:
        ms = statistics.median(res[k])
        print(json.dumps({"cfg": k, "overrides": cfgs[k], "batch": info[k], "median_ms": round(ms, 3),
                          "sig_per_s": round(a.count / ms * 1e3, 1), "all_ms": [round(x, 2) for x in res[k]]}))


if __name__ == "__main__":
    main()
