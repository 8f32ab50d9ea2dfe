#!/bin/bash
# msg_prep in registers (MGF1 first block once, digest bits from registers, by-value out-of-line compression),
# auto sharing needs >= 2 messages per key: suite, latency table, verify rate, bench.
OUT=gpurun_out/r02ad; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest.txt 2>&1; tail -2 $OUT/pytest.txt
timeout 600 python tools/latency_probe.py > $OUT/latency.txt 2>&1; cut -c1-110 $OUT/latency.txt
timeout 600 python tools/verify_rate.py > $OUT/verify.txt 2>&1; cat $OUT/verify.txt
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
python - <<'PY'
import json
d=json.loads(open("gpurun_out/r02ad/bench.json").read().strip().splitlines()[-1])
print(d["value"], d["e2e"]["value"], d["roofline"]["frac"], d["cpu_baseline"]["value"], d["launch_latency"]["e2e_small_batch_us"], d["kernel_ms_serial"])
for k,o in d["other_sets"].items(): print(k, o["value"], o["e2e"]["value"], o["roofline"]["frac"], o["launch_latency"]["e2e_small_batch_us"])
PY
