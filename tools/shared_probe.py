"""Batch time with and without subtree sharing, per set (device events, serial and graph mode)."""

from __future__ import annotations

import json
import random
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import paper_2512_23969_b200 as hs  # noqa: E402
from paper_2512_23969_b200.engine import pack_messages  # noqa: E402

eng = hs.get_engine(0)
for set_id, count in (("128f", 4096), ("192f", 4096), ("256f", 4096), ("128f", 16384)):
    p = hs.derive(set_id)
    rng = random.Random(2512_23969)
    sk = eng.keygen_batch(set_id, [rng.randbytes(3 * p.n)])[0]
    eng.upload_keys(set_id, sk)
    msgs = [rng.randbytes(32) for _ in range(count)]
    top = 3 if set_id == "256f" else 4
    row = {"set": set_id, "count": count}
    for L in range(top + 1):
        eng.set_config(set_id, shared_layers=L, shared_auto=False)
        blob, offs = pack_messages(msgs)
        eng.stage(set_id, blob, offs, count)
        eng.bench_run(set_id, count, 2, 0, 0)
        g = sorted(eng.bench_run(set_id, count, 5, 0, 0))[2]
        eng.bench_run(set_id, count, 1, 1, 0)
        row[f"L{L}"] = {"graph_ms": round(g, 3), "serial": {k: round(v, 3) for k, v in eng.timings().items()}}
    eng.set_config(set_id, shared_layers=top, shared_auto=True)
    for T in (1, 2, 4, 8):
        eng.set_config(set_id, streams=T)
        blob, offs = pack_messages(msgs)
        eng.stage(set_id, blob, offs, count)
        eng.bench_run(set_id, count, 2, 0, 0)
        row[f"T{T}"] = sorted(eng.bench_run(set_id, count, 5, 0, 0))[2]
    print(json.dumps(row), flush=True)
