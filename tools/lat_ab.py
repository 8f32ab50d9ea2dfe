"""Interleaved A/B of library builds on small-batch latency (and one large
batch): each round runs tools/latency_probe.py once per library in its own
process (HERO_SIGN_LIB), then prints per (set, count) the median device graph
time and public-call wall time of every library.

    python tools/lat_ab.py --libs a.so,b.so [--sets 128f,192f,256f] [--counts 1,4,16,64,4096] [--rounds 3]
"""

from __future__ import annotations

import argparse
import collections
import json
import os
import statistics
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--libs", required=True)
    ap.add_argument("--sets", default="128f,192f,256f")
    ap.add_argument("--counts", default="1,4,16,64,4096")
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    libs = a.libs.split(",")
    dev = collections.defaultdict(list)
    wall = collections.defaultdict(list)
    for _ in range(a.rounds):
        for lib in libs:
            env = dict(os.environ, HERO_SIGN_LIB=str(Path(lib).resolve()))
            out = subprocess.run([sys.executable, str(ROOT / "tools/latency_probe.py"), "--sets", a.sets,
                                  "--counts", a.counts, "--reps", str(a.reps)],
                                 env=env, capture_output=True, text=True, check=True).stdout
            for line in out.splitlines():
                if line.startswith("{"):
                    d = json.loads(line)
                    dev[(lib, d["set"], d["count"])].append(d["device_graph_us"])
                    wall[(lib, d["set"], d["count"])].append(d["api_wall_us"])
    for set_id in a.sets.split(","):
        for count in [int(c) for c in a.counts.split(",")]:
            row = {"set": set_id, "count": count}
            for lib in libs:
                name = Path(lib).stem.replace("libherosign_", "")
                row[name] = {"device_us": round(statistics.median(dev[(lib, set_id, count)]), 1),
                             "api_us": round(statistics.median(wall[(lib, set_id, count)]), 1)}
            print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
