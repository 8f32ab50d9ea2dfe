#!/bin/bash
# sub-batch weights 4,..,4,1 (current) vs 8,..,8,1: end to end, interleaved, per set at the bench sizes.
OUT=gpurun_out/r02au; mkdir -p $OUT
for s in "128f 4096" "192f 16384" "256f 16384"; do set -- $s
  timeout 900 python tools/ab_e2e.py --libs paper_2512_23969_b200/libherosign_b200.so,paper_2512_23969_b200/libherosign_w8.so --set $1 --count $2 --rounds 3 >> $OUT/ab.txt 2>&1
done
cat $OUT/ab.txt
