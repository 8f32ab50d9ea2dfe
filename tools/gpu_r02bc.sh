#!/bin/bash
# TREE_Sign DRAM traffic per message on the final code (thread-local Merkle levels), then the bench line.
OUT=gpurun_out/r02bc; mkdir -p $OUT
for s in 128f 192f 256f; do
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k 'regex:tree_(chain|leaf|merkle|root)' --csv python tools/ncu_target.py --set $s --count 4096 --runs 1 --mode 1 > $OUT/traffic_$s.csv 2> $OUT/traffic_$s.err
done
python tools/tree_traffic.py --count 4096 --out $OUT/tree_traffic.json 128f=$OUT/traffic_128f.csv 192f=$OUT/traffic_192f.csv 256f=$OUT/traffic_256f.csv > $OUT/tt.log 2>&1; tail -12 $OUT/tt.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
python - <<'PY'
import json
d=json.loads(open("gpurun_out/r02bc/bench.json").read().strip().splitlines()[-1])
print(d["value"], d["e2e"]["value"], d["roofline"])
PY
