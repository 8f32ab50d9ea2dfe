#!/bin/bash
# Per-stage serial times vs graph time of small batches (default and one-tree FORS CTAs).
OUT=gpurun_out/r02w; mkdir -p $OUT
for s in 128f 192f 256f; do
timeout 300 python tools/stage_times.py --set $s --counts 1,4,16 --cfg base='{}' --cfg tiny0='{"fors_trees_per_set": 1, "fors_sets_fused": 1}' >> $OUT/stages.txt 2>&1
done
cat $OUT/stages.txt
