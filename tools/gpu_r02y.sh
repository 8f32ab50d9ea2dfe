#!/bin/bash
# overlap 0 vs 1 crossover for 192f / 256f between 1024 and 16384 messages.
OUT=gpurun_out/r02y; mkdir -p $OUT
for s in 192f 256f; do
  timeout 900 python tools/small_batch_sweep.py --set $s --counts 1536,2048,3072,4096,6144,8192,16384 --reps 6 --rounds 2 \
    --cfg ov0='{"overlap": false}' --cfg ov1='{"overlap": true}' >> $OUT/sweep.txt 2>&1
done
cat $OUT/sweep.txt | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(d['set'], d['count'], d['cfg'], d['median_us'], d['bytes_equal'])
    else: print(l.rstrip())"
