#!/bin/bash
# Small batches with the batch-size rules on: TREE_Sign shape (split 1: warp-shuffle Merkle) and native SHA path for TREE.
OUT=gpurun_out/r02aa; mkdir -p $OUT
for s in 128f 192f 256f; do
  timeout 600 python tools/small_batch_sweep.py --set $s --counts 1,4,16,64,256 --reps 10 \
    --cfg base='{}' --cfg ts1='{"tree_split": 1}' \
    --cfg natT='{"variant": {"TREE_Sign": 0}}' --cfg ts1_natT='{"tree_split": 1, "variant": {"TREE_Sign": 0}}' \
    --cfg natP='{"variant": {"host": 1}}' >> $OUT/sweep.txt 2>&1
done
cat $OUT/sweep.txt | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(d['set'], d['count'], d['cfg'], d['median_us'], d['bytes_equal'])
    else: print(l.rstrip())"
