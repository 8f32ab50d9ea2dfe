#!/bin/bash
# verify throughput A/B: HEAD (compact-loop / by-pointer prep compression) vs working tree, 16384 and 65536 signatures.
OUT=gpurun_out/r02ae; mkdir -p $OUT
for r in 1 2; do
for lib in paper_2512_23969_b200/libherosign_old.so paper_2512_23969_b200/libherosign_b200.so; do
  for c in 16384 65536; do
    echo "$lib $c $(HERO_SIGN_LIB=$lib timeout 600 python tools/verify_rate.py --count $c --reps 3 | tr '\n' ' ')" >> $OUT/verify_ab.txt
  done
done
done
cat $OUT/verify_ab.txt
