#!/bin/bash
# Session-3 check of HEAD on a fresh box (suite, smoke, bench, reference arm) and a 16-mask SHA-path sweep
# of the real kernels (tree_split 2) on the round-2 build (sweep library built on the box: too large to push).
OUT=gpurun_out/r02r; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest.txt 2>&1; tail -2 $OUT/pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1; tail -1 $OUT/smoke.txt
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
python - <<'PY'
import json
d=json.loads(open("gpurun_out/r02r/bench.json").read().strip().splitlines()[-1])
print(d["value"], d["e2e"]["value"], d["roofline"]["frac"], d["cpu_baseline"]["value"])
for k,o in d["other_sets"].items(): print(k, o["value"], o["e2e"]["value"], o["roofline"]["frac"])
PY
(cd paper_2512_23969_b200/csrc && timeout 900 make -j$(nproc) MASKS=248,184,216,104,254,253,249,250,190,62,126,232,236,105,189,122 BUILD=../../build/sweep OUT=../libherosign_sweep.so > /dev/null 2>&1)
HERO_SIGN_LIB=paper_2512_23969_b200/libherosign_sweep.so timeout 1500 python tools/variant_sweep.py --count 4096 --reps 5 --tree-split 2 > $OUT/variant_sweep.txt 2>&1
cat $OUT/variant_sweep.txt
