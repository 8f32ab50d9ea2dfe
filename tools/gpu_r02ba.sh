#!/bin/bash
OUT=gpurun_out/r02ba; mkdir -p $OUT
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
python - <<'PY'
import json
d=json.loads(open("gpurun_out/r02ba/bench.json").read().strip().splitlines()[-1])
print(d["value"], d["e2e"]["value"], d["roofline"]["frac"], d["launch_latency"]["e2e_small_batch_us"], d["launch_latency"]["device_small_batch_us"])
for k,o in d["other_sets"].items(): print(k, o["value"], o["launch_latency"]["e2e_small_batch_us"], o["launch_latency"].get("device_small_batch_us"))
PY
tail -3 $OUT/bench.err
