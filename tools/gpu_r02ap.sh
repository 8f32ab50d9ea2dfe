#!/bin/bash
# Per-call e2e of 65,536-message mixed-key calls (128f), with / without a verify between calls: old vs current library.
OUT=gpurun_out/r02ap; mkdir -p $OUT
for v in "" "--verify"; do
  HERO_SIGN_LIB=paper_2512_23969_b200/libherosign_old.so HERO_SIGN_CONFIG=paper_2512_23969_b200/old_tuned.json timeout 600 python tools/e2e_calls.py $v >> $OUT/calls.txt 2>&1
  timeout 600 python tools/e2e_calls.py $v >> $OUT/calls.txt 2>&1
done
cat $OUT/calls.txt
