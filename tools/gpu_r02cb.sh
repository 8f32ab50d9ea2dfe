#!/bin/bash
# mx248p4 (mask 1272) replaces mx184 in the shipped path list; 256f FORS_Sign on it.
# Interleaved batch A/B (FORS path 2 = mx248 vs 5 = mx248p4), then suite + smoke + bench.
OUT=gpurun_out/r02cb; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/smi.txt
V2='{"variant": {"FORS_Sign": 2, "TREE_Sign": 2, "WOTS_Sign": 0}}'
V5='{"variant": {"FORS_Sign": 5, "TREE_Sign": 2, "WOTS_Sign": 0}}'
timeout 900 python tools/ab_config.py --set 256f --count 16384 --a "$V2" --b "$V5" > $OUT/ab_fors256.txt 2>&1; tail -4 $OUT/ab_fors256.txt
V3='{"variant": {"FORS_Sign": 3, "TREE_Sign": 2, "WOTS_Sign": 0}}'
timeout 600 python tools/ab_config.py --set 192f --count 16384 --a "$V3" --b "$V5" > $OUT/ab_fors192.txt 2>&1; tail -4 $OUT/ab_fors192.txt
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest.txt 2>&1; tail -2 $OUT/pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1; tail -1 $OUT/smoke.txt
timeout 900 python bench.py --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err
python - <<'PY'
import json
d=json.loads(open("gpurun_out/r02cb/bench.json").read().strip().splitlines()[-1])
print(d["value"], d["e2e"]["value"], d["roofline"]["frac"], d["clocks"])
for k,o in d["other_sets"].items(): print(k, o["value"], o["e2e"]["value"], o["roofline"]["frac"])
PY
