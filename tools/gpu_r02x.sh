#!/bin/bash
# Small batches: overlap on/off x one-tree FORS CTAs (192f/256f ship overlap 0), counts up to 1024.
OUT=gpurun_out/r02x; mkdir -p $OUT
for s in 192f 256f 128f; do
  timeout 600 python tools/small_batch_sweep.py --set $s --counts 1,4,16,64,128,256,1024 --reps 10 \
    --cfg base='{}' --cfg ov1='{"overlap": true}' \
    --cfg tiny_ov0='{"fors_trees_per_set": 1, "fors_sets_fused": 1, "overlap": false}' \
    --cfg tiny_ov1='{"fors_trees_per_set": 1, "fors_sets_fused": 1, "overlap": true}' >> $OUT/sweep.txt 2>&1
done
cat $OUT/sweep.txt | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(d['set'], d['count'], d['cfg'], d['median_us'], d['bytes_equal'])
    else: print(l.rstrip())"
