"""Time FORS_Sign / TREE_Sign / WOTS_Sign under every compiled SHA-256 path
(engine.variants(); HERO_SIGN_LIB selects a sweep build) for each parameter set, with the set's current layout.

    python tools/variant_sweep.py [--count 4096] [--reps 5]
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import paper_2512_23969_b200 as hs  # noqa: E402
from paper_2512_23969_b200.engine import variants  # noqa: E402
from paper_2512_23969_b200.tuner import _kernel_ms, _synthetic, _trimmed_mean  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--count", type=int, default=4096)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--sets", default="128f,192f,256f")
    ap.add_argument("--kernels", default="TREE_Sign,FORS_Sign")
    ap.add_argument("--tree-split", default="1", help="comma list of tree_split values to time TREE_Sign under")
    a = ap.parse_args()
    eng = hs.get_engine(0)
    names = variants()
    out = {}
    for set_id in a.sets.split(","):
        _synthetic(eng, set_id, a.count)
        base = eng.config(set_id)
        res = {}
        try:
            for kernel in a.kernels.split(","):
                splits = [int(x) for x in a.tree_split.split(",")] if kernel == "TREE_Sign" else [1]
                for ts in splits:
                    key = f"{kernel}/split{ts}" if kernel == "TREE_Sign" else kernel
                    for v, name in enumerate(names):
                        var = dict(base["variant"])
                        var[kernel] = v
                        eng.set_config(set_id, variant=var, wots_from_tree=True, tree_split=int(ts))
                        res.setdefault(key, {})[name] = round(
                            _trimmed_mean(_kernel_ms(eng, set_id, a.count, kernel, a.reps)), 4)
        finally:
            eng.set_config(set_id, **base)
        out[set_id] = res
        print(set_id, json.dumps(res), flush=True)
    return out


if __name__ == "__main__":
    main()
