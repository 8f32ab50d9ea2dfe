#!/bin/bash
# msg_prep phase cycle counts for a 1-message batch (trace build).
OUT=gpurun_out/r02bh; mkdir -p $OUT
for s in 128f 192f 256f; do
  HERO_SIGN_LIB=paper_2512_23969_b200/libherosign_trace.so timeout 300 python tools/ncu_target.py --set $s --count 1 --runs 4 --mode 0 2>&1 | grep -v timings >> $OUT/trace.txt
done
cat $OUT/trace.txt
