#!/bin/bash
# Small-graph SHA path: latency-bound graphs (a few warps per SM) run each compression as a lone
# dependent chain, where the native path is ~15 % faster than Mx<248> (profiles/r02t_lat_probe.txt).
OUT=gpurun_out/r02ce; mkdir -p $OUT
for s in 128f 192f 256f; do
  case $s in 128f) F=2;; 192f) F=3;; 256f) F=5;; esac
  timeout 600 python tools/small_batch_sweep.py --set $s --counts 1,4,16,64 --reps 30 --rounds 3 \
    --cfg base='{}' \
    --cfg tree_native="{\"variant\": {\"FORS_Sign\": $F, \"TREE_Sign\": 0, \"WOTS_Sign\": 0}}" \
    --cfg fors_native='{"variant": {"FORS_Sign": 0, "TREE_Sign": 2, "WOTS_Sign": 0}}' \
    --cfg both_native='{"variant": {"FORS_Sign": 0, "TREE_Sign": 0, "WOTS_Sign": 0}}' \
    --cfg both_fast='{"variant": {"FORS_Sign": 1, "TREE_Sign": 1, "WOTS_Sign": 0}}' >> $OUT/small_paths.txt 2>&1
done
cat $OUT/small_paths.txt
