"""Run the on-device Tree Tuning + SHA-path selection for every set; write the config JSON.

    python tools/tune_all.py [--out gpurun_out/tuning.json] [--count 2048]
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import paper_2512_23969_b200 as hs  # noqa: E402
from paper_2512_23969_b200.config import TuningConfig  # noqa: E402
from paper_2512_23969_b200.tuner import tune_on_device  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/tuning.json")
    ap.add_argument("--count", type=int, default=4096)
    ap.add_argument("--top", type=int, default=12)
    a = ap.parse_args()
    eng = hs.get_engine(0)
    report = {}
    for set_id in ("128f", "192f", "256f"):
        r = tune_on_device(eng, set_id, count=a.count, top=a.top)
        report[set_id] = r
        print(set_id, json.dumps({"best": r["best_layout"], "variants": r["variants"], "variant_ms": r["variant_ms"],
                                  "streams_ms": r["streams_ms"]}), flush=True)
    cfg = TuningConfig.from_engine(eng)
    cfg.save(a.out)
    Path(a.out).with_suffix(".report.json").write_text(json.dumps(report, indent=1, default=str))


if __name__ == "__main__":
    main()
