#!/bin/bash
# Final code check: suite, smoke, latency table, bench + reference arm.
OUT=gpurun_out/r02bi; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest.txt 2>&1; tail -2 $OUT/pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1; tail -1 $OUT/smoke.txt
timeout 600 python tools/latency_probe.py > $OUT/latency.txt 2>&1; cut -c1-150 $OUT/latency.txt
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
python - <<'PY'
import json
d=json.loads(open("gpurun_out/r02bi/bench.json").read().strip().splitlines()[-1])
print(d["value"], d["e2e"]["value"], d["roofline"]["frac"], d["launch_latency"]["e2e_small_batch_us"], d["launch_latency"]["device_small_batch_us"], d["clocks"])
for k,o in d["other_sets"].items(): print(k, o["value"], o["e2e"]["value"], o["roofline"]["frac"], o["launch_latency"]["e2e_small_batch_us"], o["launch_latency"]["device_small_batch_us"])
r=json.loads(open("gpurun_out/r02bi/bench_ref.json").read().strip().splitlines()[-1]); print("ref", r["value"])
PY
