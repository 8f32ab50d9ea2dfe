"""Interleaved A/B of library builds on one GPU: per set, the serial-mode kernel
times (FORS_Sign, TREE_Sign) and the graph-mode batch time, each lib in its own
process (HERO_SIGN_LIB), rounds interleaved.

    python tools/lib_ab.py --libs paper_2512_23969_b200/libherosign_b200.so,X.so \
        --sets 192f:16384,256f:16384 [--rounds 3] [--reps 5]
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
CHILD = r'''
import json, sys
sys.path.insert(0, {root!r})
import paper_2512_23969_b200 as hs
from paper_2512_23969_b200.tuner import _synthetic, _kernel_ms
eng = hs.get_engine(0)
out = {{}}
for spec in {sets!r}:
    set_id, count = spec.split(":"); count = int(count)
    _synthetic(eng, set_id, count)
    eng.bench_run(set_id, count, 2, 0, 256 << 20)
    batch = eng.bench_run(set_id, count, {reps}, 0, 256 << 20)
    k = {{kn: _kernel_ms(eng, set_id, count, kn, {reps}) for kn in ("FORS_Sign", "TREE_Sign")}}
    out[set_id] = {{"batch": batch, **k}}
print(json.dumps(out))
'''


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--libs", required=True)
    ap.add_argument("--sets", default="128f:4096,192f:16384,256f:16384")
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    libs = a.libs.split(",")
    sets = a.sets.split(",")
    code = CHILD.format(root=str(ROOT), sets=sets, reps=a.reps)
    res = {lib: {} for lib in libs}
    for _ in range(a.rounds):
        for lib in libs:
            env = dict(os.environ, HERO_SIGN_LIB=str(Path(lib).resolve()))
            p = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
            if p.returncode != 0:
                print(f"{lib}: failed\n{p.stderr[-2000:]}", flush=True)
                continue
            for sid, d in json.loads(p.stdout.strip().splitlines()[-1]).items():
                for k, v in d.items():
                    res[lib].setdefault(sid, {}).setdefault(k, []).extend(v)
    for lib, per in res.items():
        for sid, d in per.items():
            line = "  ".join(f"{k} {statistics.median(v):.3f} ms" for k, v in d.items())
            print(f"{Path(lib).name:32s} {sid:5s} {line}", flush=True)


if __name__ == "__main__":
    main()
