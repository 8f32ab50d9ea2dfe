"""Device latency of small batches under alternative engine configs, with the
bytes of every config checked against the default's.

    python tools/small_batch_sweep.py --set 128f --counts 1,4,16,64 \
        --cfg base='{}' --cfg tiny='{"fors_trees_per_set": 1, "fors_sets_fused": 1, "fors_cta_levels": 6}'
"""

from __future__ import annotations

import argparse
import json
import random
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import paper_2512_23969_b200 as hs  # noqa: E402
from paper_2512_23969_b200.engine import pack_messages  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--set", dest="set_id", default="128f")
    ap.add_argument("--counts", default="1,4,16,64")
    ap.add_argument("--cfg", action="append", default=[], help="name=json overrides")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--rounds", type=int, default=2)
    a = ap.parse_args()
    eng = hs.get_engine(0)
    p = hs.derive(a.set_id)
    base = eng.config(a.set_id)
    cfgs = dict(c.split("=", 1) for c in (a.cfg or ["base={}"]))
    cfgs = {k: json.loads(v) for k, v in cfgs.items()}
    rng = random.Random(2512_23969)
    sk = eng.keygen_batch(a.set_id, [rng.randbytes(3 * p.n)])[0]
    eng.upload_keys(a.set_id, sk)
    for count in [int(c) for c in a.counts.split(",")]:
        msgs = [rng.randbytes(32) for _ in range(count)]
        blob, offs = pack_messages(msgs)
        eng.set_config(a.set_id, **base)
        ref = eng.sign_batch(a.set_id, msgs)
        res = {k: [] for k in cfgs}
        ok = {}
        try:
            for _ in range(a.rounds):
                for k, c in cfgs.items():
                    eng.set_config(a.set_id, **{**base, **c})
                    ok[k] = eng.sign_batch(a.set_id, msgs) == ref
                    eng.stage(a.set_id, blob, offs, count)
                    eng.bench_run(a.set_id, count, 3, 0)
                    res[k] += eng.bench_run(a.set_id, count, a.reps, 0)
        finally:
            eng.set_config(a.set_id, **base)
        for k in cfgs:
            print(json.dumps({"set": a.set_id, "count": count, "cfg": k, "overrides": cfgs[k],
                              "median_us": round(1e3 * statistics.median(res[k]), 1),
                              "min_us": round(1e3 * min(res[k]), 1), "bytes_equal": ok[k]}), flush=True)


if __name__ == "__main__":
    main()
