"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into per-kernel shares.

    python tools/launch_summary.py gpurun_out/launches.csv > profiles/r01_launches.md
"""

from __future__ import annotations

import collections
import csv
import sys


def main(path: str) -> None:
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr, data = rows[hi], rows[hi + 1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3}
    agg = collections.defaultdict(list)
    for r in data:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("void ", "").replace("hs::", "")
        agg[name].append(float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0))
    tot = sum(sum(v) for v in agg.values())
    print("| kernel | launches | avg ms | share |")
    print("|---|---|---|---|")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"| `{k}` | {len(v)} | {sum(v) / len(v):.3f} | {100 * sum(v) / tot:.1f}% |")


if __name__ == "__main__":
    main(sys.argv[1])
