#!/bin/bash
# 128f tree_small_batch 64 (shipped) vs 16 (the 4,096-message tuning run's pick), 16-64 message graphs.
OUT=gpurun_out/r02cm; mkdir -p $OUT
timeout 600 python tools/small_batch_sweep.py --set 128f --counts 16,24,32,48,64 --reps 30 --rounds 3 \
  --cfg ts64='{}' --cfg ts16='{"tree_small_batch": 16}' > $OUT/tsmall.txt 2>&1; cat $OUT/tsmall.txt
