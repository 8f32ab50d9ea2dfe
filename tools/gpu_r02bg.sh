#!/bin/bash
# 256f small graphs after the TREE-path latency work: FORS shape (one tree per CTA, in-CTA levels) and per-stage times.
OUT=gpurun_out/r02bg; mkdir -p $OUT
timeout 900 python tools/small_batch_sweep.py --set 256f --counts 1,4,16,64 --reps 10 \
  --cfg base='{}' --cfg tiny='{"fors_small_batch": 64}' --cfg tinyL='{"fors_small_batch": 64, "fors_cta_levels": 9}' \
  --cfg L9='{"fors_cta_levels": 9}' --cfg L0='{"fors_cta_levels": 0}' > $OUT/sweep256.txt 2>&1
timeout 900 python tools/small_batch_sweep.py --set 192f --counts 1,4,16,64 --reps 10 \
  --cfg base='{}' --cfg tinyL='{"fors_cta_levels": 8}' --cfg small0='{"fors_small_batch": 0}' > $OUT/sweep192.txt 2>&1
timeout 900 python tools/small_batch_sweep.py --set 128f --counts 1,4,16,64 --reps 10 \
  --cfg base='{}' --cfg tinyL='{"fors_cta_levels": 6}' > $OUT/sweep128.txt 2>&1
timeout 300 python tools/stage_times.py --set 256f --counts 1,16 >> $OUT/stages.txt 2>&1
cat $OUT/sweep*.txt | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(d['set'], d['count'], d['cfg'], d['median_us'], d['bytes_equal'])"
cat $OUT/stages.txt
