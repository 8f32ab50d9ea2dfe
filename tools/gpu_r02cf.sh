#!/bin/bash
# Re-check of r02ce on another box: 128f 1-4 message graphs with the FORS / TREE SHA path varied.
OUT=gpurun_out/r02cf; mkdir -p $OUT
timeout 600 python tools/small_batch_sweep.py --set 128f --counts 1,2,4 --reps 50 --rounds 5 \
  --cfg base='{}' \
  --cfg fors_native='{"variant": {"FORS_Sign": 0, "TREE_Sign": 2, "WOTS_Sign": 0}}' \
  --cfg fors_fast='{"variant": {"FORS_Sign": 1, "TREE_Sign": 2, "WOTS_Sign": 0}}' \
  --cfg tree_fast='{"variant": {"FORS_Sign": 2, "TREE_Sign": 1, "WOTS_Sign": 0}}' \
  --cfg both_fast='{"variant": {"FORS_Sign": 1, "TREE_Sign": 1, "WOTS_Sign": 0}}' > $OUT/small_paths.txt 2>&1
timeout 300 python tools/latency_probe.py --counts 1,4 > $OUT/latency_probe.txt 2>&1 || true
cat $OUT/small_paths.txt
