#!/bin/bash
# Pipe balancing across concurrent kernels: FORS_Sign SHA path (0 native, 1 fast, 2 mx248, 3 mx232, 4 mx104, 5 mx184)
# in the overlapped batch graph (FORS || TREE), graph device time.
OUT=gpurun_out/r02bd; mkdir -p $OUT
timeout 900 python tools/small_batch_sweep.py --set 128f --counts 4096 --reps 6 --rounds 2 \
  --cfg v2='{"variant": {"FORS_Sign": 2}}' --cfg v0='{"variant": {"FORS_Sign": 0}}' --cfg v1='{"variant": {"FORS_Sign": 1}}' \
  --cfg v3='{"variant": {"FORS_Sign": 3}}' --cfg v4='{"variant": {"FORS_Sign": 4}}' --cfg v5='{"variant": {"FORS_Sign": 5}}' >> $OUT/sweep.txt 2>&1
timeout 1200 python tools/small_batch_sweep.py --set 192f --counts 16384 --reps 3 --rounds 1 \
  --cfg ov0_v3='{"overlap": 0, "variant": {"FORS_Sign": 3}}' --cfg ov1_v3='{"overlap": 1, "variant": {"FORS_Sign": 3}}' \
  --cfg ov1_v1='{"overlap": 1, "variant": {"FORS_Sign": 1}}' --cfg ov1_v0='{"overlap": 1, "variant": {"FORS_Sign": 0}}' >> $OUT/sweep.txt 2>&1
cat $OUT/sweep.txt
