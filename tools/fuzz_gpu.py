"""Randomised GPU-vs-oracle soak test: random parameter set, batch size,
message lengths, key count, opt_rand mix and engine configuration (FORS
layout from every feasible candidate, in-CTA levels, TREE_Sign shape, SHA
paths, sub-batches, stream overlap / thresholds, small-graph rules, subtree
sharing, chunk size) per iteration; every signature is compared with the
oracle and verified on the GPU.  Prints the seed of any failure.

    python tools/fuzz_gpu.py [--minutes 10] [--seed 1]
"""

from __future__ import annotations

import argparse
import json
import random
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

import oracle  # noqa: E402  (checker)

import paper_2512_23969_b200 as hs  # noqa: E402
from paper_2512_23969_b200.engine import variants  # noqa: E402
from paper_2512_23969_b200.tuner import device_candidates  # noqa: E402


def random_config(rng: random.Random, p, cands, nvar: int) -> dict:
    c = rng.choice(cands)
    cfg = {"fors_trees_per_set": c.trees_per_set, "fors_sets_fused": c.sets_fused, "fors_relax": c.relax,
           "fors_cta_levels": rng.choice([-1, p.log_t, rng.randrange(1 if c.relax else 0, p.log_t + 1)]),
           "tree_split": rng.choice([0, 1, 2, 2]),
           "variant": {k: rng.randrange(nvar) for k in ("FORS_Sign", "TREE_Sign", "WOTS_Sign", "host")},
           "streams": rng.choice([1, 2, 3, 4, 8]),
           "overlap": rng.choice([0, 1, 2, 16, 100, 1536]),
           "fors_small_batch": rng.choice([0, 0, 4, 16, 64]),
           "tree_small_batch": rng.choice([0, 0, 4, 16, 64]),
           "wots_from_tree": rng.random() < 0.85,
           "shared_auto": rng.random() < 0.5,
           "chunk": rng.choice([64, 256, 1024, 16384])}
    top = 4 if p.id == "256f" else 6
    cfg["shared_layers"] = rng.randrange(top + 1)
    return cfg


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--minutes", type=float, default=10.0)
    ap.add_argument("--seed", type=int, default=1)
    a = ap.parse_args()
    eng = hs.get_engine(0)
    nvar = len(variants())
    smem = eng.device_info()["smem_optin"]
    cands = {s: device_candidates(hs.derive(s), smem, alpha=0.0) for s in ("128f", "192f", "256f")}
    base = {s: eng.config(s) for s in cands}
    oracle.build()
    t_end = time.time() + 60 * a.minutes
    it = fails = sigs_checked = 0
    while time.time() < t_end:
        seed = a.seed * 1_000_003 + it
        rng = random.Random(seed)
        set_id = rng.choice(["128f", "128f", "192f", "256f"])
        p = hs.derive(set_id)
        nkeys = rng.choice([1, 1, 2, 3])
        sks = [oracle.keygen(set_id, rng.randbytes(3 * p.n)) for _ in range(nkeys)]
        count = rng.choice([1, 2, 3, 5, 17, 31, 64, 65, 130, 257, 300])
        msgs = [rng.randbytes(rng.choice([0, 1, 31, 32, 33, 64, 65, 100, 200])) for _ in range(count)]
        kidx = [rng.randrange(nkeys) for _ in range(count)]
        opts = [rng.randbytes(p.n) if rng.random() < 0.3 else None for _ in range(count)]
        cfg = random_config(rng, p, cands[set_id], nvar)
        try:
            eng.set_config(set_id, **cfg)
            eng.upload_keys(set_id, sks)
            got = eng.sign_batch(set_id, msgs, key_idx=kidx, opt_rand=opts)
            orand = b"".join(o if o is not None else sks[kidx[i]][2 * p.n:3 * p.n] for i, o in enumerate(opts))
            ref, _ = oracle.sign_many(set_id, b"".join(sks), kidx, msgs, orand)
            bad = [i for i in range(count) if got[i] != ref[i]]
            ok = eng.verify_batch(set_id, [sk[2 * p.n:] for sk in sks], msgs, got, key_idx=kidx)
            if bad or not all(ok):
                fails += 1
                print(json.dumps({"FAIL": seed, "set": set_id, "count": count, "bad": bad[:5],
                                  "verify_fail": [i for i, v in enumerate(ok) if not v][:5], "cfg": cfg}), flush=True)
            sigs_checked += count
        finally:
            eng.set_config(set_id, **base[set_id])
        it += 1
    print(json.dumps({"iterations": it, "signatures_checked": sigs_checked, "failures": fails,
                      "minutes": a.minutes, "seed": a.seed}))
    sys.exit(1 if fails else 0)


if __name__ == "__main__":
    main()
