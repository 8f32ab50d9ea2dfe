#!/bin/bash
# Batch-size rules (fors_small_batch, overlap threshold) + latency kernel changes: suite, latency table, bench.
OUT=gpurun_out/r02z; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest.txt 2>&1; tail -2 $OUT/pytest.txt
timeout 600 python tools/latency_probe.py > $OUT/latency.txt 2>&1; cat $OUT/latency.txt
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
python - <<'PY'
import json
d=json.loads(open("gpurun_out/r02z/bench.json").read().strip().splitlines()[-1])
print(d["value"], d["e2e"]["value"], d["roofline"]["frac"], d["cpu_baseline"]["value"], d["launch_latency"]["e2e_small_batch_us"])
for k,o in d["other_sets"].items(): print(k, o["value"], o["e2e"]["value"], o["roofline"]["frac"], o["launch_latency"]["e2e_small_batch_us"])
PY
