"""A/B end-to-end (public API, pinned host buffers, H2D + sign + D2H) timing of
two library builds, interleaved in separate processes on the same GPU:
    python tools/ab_e2e.py --libs A.so,B.so --set 128f --count 4096"""

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
import json, random, sys, time
sys.path.insert(0, {root!r})
import numpy as np
import paper_2512_23969_b200 as hs
from paper_2512_23969_b200.engine import PinnedBuffer, pack_messages
from paper_2512_23969_b200.params import derive
set_id, count, steps = {set_id!r}, {count}, {steps}
p = derive(set_id)
rng = random.Random(2512_23969)
seed = rng.randbytes(3 * p.n)
msgs = [rng.randbytes(32) for _ in range(count)]
eng = hs.get_engine(0)
sk = eng.keygen_batch(set_id, [seed])[0]
eng.upload_keys(set_id, sk)
blob, offs = pack_messages(msgs)
hb = PinnedBuffer(len(blob)); hb.array()[:len(blob)] = np.frombuffer(blob, dtype=np.uint8)
ho = PinnedBuffer(offs.nbytes); ho.array(np.uint64)[:] = offs
out = PinnedBuffer(count * p.sig_bytes)
for _ in range(3):
    eng.sign_into(set_id, hb.ptr, ho.array(np.uint64), count, out.ptr)
t = []
for _ in range(steps):
    t0 = time.perf_counter(); eng.sign_into(set_id, hb.ptr, ho.array(np.uint64), count, out.ptr); t.append(time.perf_counter() - t0)
print(json.dumps(t))
'''


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--libs", required=True)
    ap.add_argument("--set", dest="set_id", default="128f")
    ap.add_argument("--count", type=int, default=4096)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--rounds", type=int, default=3)
    a = ap.parse_args()
    libs = a.libs.split(",")
    res = {lib: [] for lib in libs}
    code = CHILD.format(root=str(ROOT), set_id=a.set_id, count=a.count, steps=a.steps)
    for _ in range(a.rounds):
        for lib in libs:
            env = dict(os.environ, HERO_SIGN_LIB=str(Path(lib).resolve()))
            outp = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, check=True)
            res[lib] += json.loads(outp.stdout.strip().splitlines()[-1])
    for lib, t in res.items():
        med = statistics.median(t)
        print(json.dumps({"lib": Path(lib).name, "set": a.set_id, "count": a.count, "median_ms": round(1e3 * med, 3),
                          "sig_per_s": round(a.count / med, 1)}))


if __name__ == "__main__":
    main()
