"""Per-message DRAM traffic of the per-message TREE_Sign kernels from ncu CSVs
-> profiles/tree_traffic.json (the bench line's roofline `traffic`).

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum -k regex:'tree_(chain|leaf|merkle|root)' \
        --csv python tools/ncu_target.py --set 128f --count 4096 --runs 1 --mode 1 > t128f.csv
    python tools/tree_traffic.py --count 4096 128f=t128f.csv 192f=t192f.csv 256f=t256f.csv
"""

from __future__ import annotations

import argparse
import csv
import io
import json
from pathlib import Path

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def kernel_bytes(path: str) -> dict:
    text = Path(path).read_text()
    start = text.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    out = {}
    for r in rows:
        if r.get("Metric Name") not in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            continue
        name = r["Kernel Name"].split("<")[0].split("(")[0].replace("void ", "").replace("hs::", "")
        v = float(r["Metric Value"].replace(",", "")) * UNIT.get(r["Metric Unit"], 1)
        out[name] = out.get(name, 0.0) + v
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--count", type=int, default=4096)
    ap.add_argument("--out", default=str(Path(__file__).resolve().parent.parent / "profiles" / "tree_traffic.json"))
    ap.add_argument("inputs", nargs="+", help="set=ncu.csv")
    a = ap.parse_args()
    res = {}
    for spec in a.inputs:
        set_id, path = spec.split("=", 1)
        kb = kernel_bytes(path)
        res[set_id] = {
            "bytes_per_launch_per_msg": int(round(sum(kb.values()) / a.count)),
            "per_kernel_bytes_per_msg": {k: int(round(v / a.count)) for k, v in sorted(kb.items())},
            "source": f"ncu dram__bytes_read.sum + dram__bytes_write.sum of the per-message TREE_Sign kernels "
                      f"({', '.join(sorted(kb))}), {a.count} msgs, tuned config, serial mode; per message: chain "
                      f"ends written once and read once, the signing-leaf stash, leaf/Merkle records",
        }
    Path(a.out).write_text(json.dumps(res, indent=1) + "\n")
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
