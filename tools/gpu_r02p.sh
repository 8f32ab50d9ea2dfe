#!/bin/bash
# GPU suite + bench with tree_split 2 everywhere and overlap off for 192f/256f.
OUT=gpurun_out/r02p; mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest.txt 2>&1; tail -2 $OUT/pytest.txt
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
python - <<'PY'
import json
d=json.loads(open("gpurun_out/r02p/bench.json").read().strip().splitlines()[-1])
print(d["value"], d["e2e"]["value"], d["roofline"]["frac"], d["cpu_baseline"]["value"])
for k,o in d["other_sets"].items(): print(k, o["value"], o["e2e"]["value"], o["roofline"]["frac"])
PY
cat $OUT/bench_ref.json | head -c 200
