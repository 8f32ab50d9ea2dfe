#!/bin/bash
# Whole FORS tree in the CTA for 1-2 message graphs (fewer graph nodes, no level-grid launches on the FORS branch).
OUT=gpurun_out/r02bm; mkdir -p $OUT
for s in "128f 6" "192f 8" "256f 9"; do set -- $s
  timeout 600 python tools/small_batch_sweep.py --set $1 --counts 1,2,3,4 --reps 20 --rounds 2 \
    --cfg base='{}' --cfg L="{\"fors_cta_levels\": $2}" >> $OUT/sweep.txt 2>&1
done
cat $OUT/sweep.txt | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(d['set'], d['count'], d['cfg'], d['median_us'], d['bytes_equal'])"
