#!/bin/bash
# 128f FORS_Sign narrow bound experiments + FORS SHA-path sweep on the narrow-kernel build (192f / 256f).
OUT=gpurun_out/r02cj; mkdir -p $OUT
timeout 900 python tools/lib_ab.py --libs paper_2512_23969_b200/libherosign_b200.so,swlibs/libhs_e384.so \
  --sets 128f:4096 --rounds 5 --reps 10 > $OUT/lib_ab_e384.txt 2>&1; cat $OUT/lib_ab_e384.txt
export HERO_SIGN_LIB=$PWD/swlibs/libhs_e256.so
timeout 600 python tools/ab_config.py --set 128f --count 4096 --rounds 5 --serial --a '{}' --b '{"fors_trees_per_set": 4, "fors_sets_fused": 8}' > $OUT/ab_e256_a.txt 2>&1; cut -c1-420 $OUT/ab_e256_a.txt
timeout 600 python tools/ab_config.py --set 128f --count 4096 --rounds 5 --serial --a '{"fors_trees_per_set": 4, "fors_sets_fused": 4}' --b '{"fors_trees_per_set": 2, "fors_sets_fused": 8}' > $OUT/ab_e256_b.txt 2>&1; cut -c1-420 $OUT/ab_e256_b.txt
unset HERO_SIGN_LIB
timeout 900 python tools/variant_sweep.py --sets 192f,256f --count 16384 --reps 3 --kernels FORS_Sign > $OUT/fors_paths.txt 2>&1; cat $OUT/fors_paths.txt
