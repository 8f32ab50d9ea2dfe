"""Per-call wall time of consecutive 65,536-message sign_into calls (mixed keys,
pinned output), optionally with a GPU verify between calls: where the
end-to-end rate of the config-5 stress goes.

    python tools/e2e_calls.py [--set 128f] [--calls 8] [--verify]
"""

from __future__ import annotations

import argparse
import json
import random
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import paper_2512_23969_b200 as hs  # noqa: E402
from paper_2512_23969_b200.engine import PinnedBuffer, pack_messages  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--set", dest="set_id", default="128f")
    ap.add_argument("--calls", type=int, default=8)
    ap.add_argument("--count", type=int, default=65536)
    ap.add_argument("--keys", type=int, default=1024)
    ap.add_argument("--verify", action="store_true")
    a = ap.parse_args()
    eng = hs.get_engine(0)
    p = hs.derive(a.set_id)
    rng = random.Random(11)
    sks = eng.keygen_batch(a.set_id, [rng.randbytes(3 * p.n) for _ in range(a.keys)])
    eng.upload_keys(a.set_id, sks)
    pks = b"".join(sk[2 * p.n:] for sk in sks)
    out = PinnedBuffer(a.count * p.sig_bytes)
    kidx = np.arange(a.count, dtype=np.uint32) % a.keys
    times = []
    try:
        for c in range(a.calls):
            blob, offs = pack_messages([rng.randbytes(32) for _ in range(a.count)])
            t0 = time.perf_counter()
            eng.sign_into(a.set_id, blob, offs, a.count, out.ptr, key_idx=kidx)
            times.append(round(1e3 * (time.perf_counter() - t0), 2))
            if a.verify:
                assert eng.verify_into(a.set_id, pks, blob, offs, a.count, out.ptr, key_idx=kidx).all()
        eng.stage(a.set_id, blob, offs, min(a.count, eng.config(a.set_id)["chunk"]), key_idx=kidx)
        n = min(a.count, eng.config(a.set_id)["chunk"])
        eng.bench_run(a.set_id, n, 1, 0, 0)
        dev = eng.bench_run(a.set_id, n, 3, 0, 0)
    finally:
        out.free()
    dev_call_ms = sum(dev) / len(dev) * a.count / n
    print(json.dumps({"set": a.set_id, "verify_between": a.verify, "call_ms": times,
                      "device_ms_per_call": round(dev_call_ms, 2),
                      "e2e_over_device_steady": round(dev_call_ms / (sum(times[1:]) / (len(times) - 1)), 4)}))


if __name__ == "__main__":
    main()
