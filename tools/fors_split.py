"""FORS_Sign (+ upper-level grids + T_k) device time per fors_cta_levels value,
for each set at its tuned layout and a few others.

    python tools/fors_split.py [--count 4096]
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import paper_2512_23969_b200 as hs  # noqa: E402
from paper_2512_23969_b200.params import derive  # noqa: E402
from paper_2512_23969_b200.tuner import _kernel_ms, _synthetic, _trimmed_mean  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--count", type=int, default=4096)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    eng = hs.get_engine(0)
    for set_id in ("128f", "192f", "256f"):
        p = derive(set_id)
        _synthetic(eng, set_id, a.count)
        base = eng.config(set_id)
        layouts = [(base["fors_trees_per_set"], base["fors_sets_fused"], base["fors_relax"]), (1, 1, False),
                   (1, 4, False), (1, 2, True)]
        res = {}
        try:
            for nt, f, rx in layouts:
                row = {}
                for lc in [-1] + list(range(1 if rx else 0, p.log_t + 1)):
                    eng.set_config(set_id, fors_trees_per_set=nt, fors_sets_fused=f, fors_relax=rx, fors_cta_levels=lc)
                    row["auto" if lc < 0 else str(lc)] = round(
                        _trimmed_mean(_kernel_ms(eng, set_id, a.count, "FORS_Sign", a.reps)), 4)
                res[f"{nt}x{f}{'R' if rx else ''}"] = row
        finally:
            eng.set_config(set_id, **base)
        print(set_id, json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
