"""Per-stage device times of one staged batch in serial mode (mode 1: msg_prep,
FORS_Sign, TREE_Sign, WOTS_Sign each between CUDA events) next to the graph
time (mode 0), under optional config overrides.

    python tools/stage_times.py --set 128f --counts 1,4 [--cfg name='{json}' ...]
"""

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
    ap.add_argument("--set", dest="set_id", default="128f")
    ap.add_argument("--counts", default="1,4,16")
    ap.add_argument("--cfg", action="append", default=[])
    ap.add_argument("--reps", type=int, default=15)
    a = ap.parse_args()
    eng = hs.get_engine(0)
    base = eng.config(a.set_id)
    cfgs = {k: json.loads(v) for k, v in (c.split("=", 1) for c in (a.cfg or ["base={}"]))}
    try:
        for count in [int(c) for c in a.counts.split(",")]:
            for name, c in cfgs.items():
                eng.set_config(a.set_id, **{**base, **c})
                _synthetic(eng, a.set_id, count)
                eng.bench_run(a.set_id, count, 3, 0)
                graph = statistics.median(eng.bench_run(a.set_id, count, a.reps, 0))
                ser = {}
                for _ in range(a.reps):
                    eng.bench_run(a.set_id, count, 1, 1)
                    for k, v in eng.timings().items():
                        ser.setdefault(k, []).append(v)
                print(json.dumps({"set": a.set_id, "count": count, "cfg": name, "graph_us": round(1e3 * graph, 1),
                                  "serial_us": {k: round(1e3 * statistics.median(v), 1) for k, v in ser.items()},
                                  "batch": eng.batch_info(a.set_id)}), flush=True)
    finally:
        eng.set_config(a.set_id, **base)


if __name__ == "__main__":
    main()
