#!/bin/bash
# verify rate vs batch size (latency-bound below the occupancy cap?)
OUT=gpurun_out/r02ar; mkdir -p $OUT
for c in 16384 65536 262144; do timeout 900 python tools/verify_rate.py --sets 128f,256f --count $c --reps 3 >> $OUT/verify_sizes.txt 2>&1; done
cat $OUT/verify_sizes.txt
