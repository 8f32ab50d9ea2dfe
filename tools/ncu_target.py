"""Minimal launcher for ncu captures: stage one synthetic batch and run it.

    python tools/ncu_target.py --set 128f --count 4096 --runs 2 [--mode 0|1]
"""

from __future__ import annotations

import argparse
import random
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import paper_2512_23969_b200 as hs  # noqa: E402
from paper_2512_23969_b200.engine import pack_messages  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--set", dest="set_id", default="128f")
    ap.add_argument("--count", type=int, default=4096)
    ap.add_argument("--runs", type=int, default=2)
    ap.add_argument("--mode", type=int, default=1)
    ap.add_argument("--variant", type=int, default=None)
    a = ap.parse_args()
    p = hs.derive(a.set_id)
    rng = random.Random(2512_23969)
    seed = rng.randbytes(3 * p.n)
    msgs = [rng.randbytes(32) for _ in range(a.count)]
    eng = hs.get_engine(0)
    if a.variant is not None:
        eng.set_config(a.set_id, variant={k: a.variant for k in ("FORS_Sign", "TREE_Sign", "WOTS_Sign", "host")})
    sk = eng.keygen_batch(a.set_id, [seed])[0]
    eng.upload_keys(a.set_id, sk)
    blob, offs = pack_messages(msgs)
    eng.stage(a.set_id, blob, offs, a.count)
    for _ in range(a.runs):
        eng.run(a.set_id, a.count, a.mode)
    eng.sync()
    print("timings", eng.timings())


if __name__ == "__main__":
    main()
