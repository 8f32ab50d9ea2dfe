#!/bin/bash
# FORS_Sign occupancy experiment: launch bound (lanes, minBlocks) = (256, 4) for 192f and (512, 2)
# for 256f (64 registers) in swlibs/libhs_fexp.so vs the shipped 768-lane bound, under the shipped
# fused-set counts and smaller ones (smem per CTA small enough for 2-4 CTAs per SM).
OUT=gpurun_out/r02cc; mkdir -p $OUT
for lib in default swlibs/libhs_fexp.so; do
  if [ $lib = default ]; then unset HERO_SIGN_LIB; else export HERO_SIGN_LIB=$PWD/$lib; fi
  echo "== $lib 256f" >> $OUT/ab.txt
  timeout 900 python tools/ab_config.py --set 256f --count 16384 --serial --a '{"fors_sets_fused": 7}' --b '{"fors_sets_fused": 4}' >> $OUT/ab.txt 2>&1
  timeout 900 python tools/ab_config.py --set 256f --count 16384 --serial --a '{"fors_sets_fused": 3}' --b '{"fors_sets_fused": 2}' >> $OUT/ab.txt 2>&1
  echo "== $lib 192f" >> $OUT/ab.txt
  timeout 900 python tools/ab_config.py --set 192f --count 16384 --serial --a '{"fors_sets_fused": 11}' --b '{"fors_sets_fused": 5}' >> $OUT/ab.txt 2>&1
  timeout 900 python tools/ab_config.py --set 192f --count 16384 --serial --a '{"fors_sets_fused": 7}' --b '{"fors_sets_fused": 4}' >> $OUT/ab.txt 2>&1
done
cut -c1-400 $OUT/ab.txt
