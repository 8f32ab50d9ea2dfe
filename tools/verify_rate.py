"""GPU verification throughput: sign `count` messages into a pinned buffer, then
time Engine.verify_into over them (public call, zero-copy from that buffer).

    python tools/verify_rate.py [--sets 128f,192f,256f] [--count 16384] [--reps 5]
"""

from __future__ import annotations

import argparse
import json
import random
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import paper_2512_23969_b200 as hs  # noqa: E402
from paper_2512_23969_b200.engine import PinnedBuffer, pack_messages  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sets", default="128f,192f,256f")
    ap.add_argument("--count", type=int, default=16384)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    eng = hs.get_engine(0)
    for set_id in a.sets.split(","):
        p = hs.derive(set_id)
        rng = random.Random(5)
        sk = eng.keygen_batch(set_id, [rng.randbytes(3 * p.n)])[0]
        eng.upload_keys(set_id, sk)
        blob, offs = pack_messages([rng.randbytes(32) for _ in range(a.count)])
        out = PinnedBuffer(a.count * p.sig_bytes)
        try:
            eng.sign_into(set_id, blob, offs, a.count, out.ptr)
            pk = sk[2 * p.n:]
            assert eng.verify_into(set_id, pk, blob, offs, a.count, out.ptr).all()
            runs = []
            for _ in range(a.reps):
                t0 = time.perf_counter()
                ok = eng.verify_into(set_id, pk, blob, offs, a.count, out.ptr)
                runs.append(time.perf_counter() - t0)
            assert ok.all()
        finally:
            out.free()
        print(json.dumps({"set": set_id, "count": a.count,
                          "verify_per_s": round(a.count / statistics.median(runs), 1)}), flush=True)


if __name__ == "__main__":
    main()
