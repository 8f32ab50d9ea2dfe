#!/bin/bash
# What is on the 1-message critical path: no shared subtrees (no memset, no shared branch), native TREE path, both.
OUT=gpurun_out/r02ac; mkdir -p $OUT
for s in 128f 192f 256f; do
  timeout 600 python tools/small_batch_sweep.py --set $s --counts 1,4 --reps 20 \
    --cfg base='{}' --cfg noshare='{"shared_layers": 0}' \
    --cfg natT='{"variant": {"FORS_Sign": 2, "TREE_Sign": 0, "WOTS_Sign": 0, "host": 0}}' >> $OUT/sweep.txt 2>&1
done
python tools/stage_times.py --set 128f --counts 1 >> $OUT/sweep.txt 2>&1
cat $OUT/sweep.txt | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(d['set'], d['count'], d.get('cfg'), d.get('median_us', d.get('graph_us')), d.get('serial_us', d.get('bytes_equal')))
    else: print(l.rstrip())"
