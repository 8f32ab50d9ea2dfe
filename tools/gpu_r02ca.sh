#!/bin/bash
# Session-4 first call: GPU suite + smoke on the restored build, then the TREE_Sign / FORS_Sign
# SHA-path sweep with masks not in the shipped list (post rotation-hoist build), real kernels.
OUT=gpurun_out/r02ca; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest.txt 2>&1; tail -2 $OUT/pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1; tail -1 $OUT/smoke.txt
for lib in default swlibs/libhs_swA.so swlibs/libhs_swB.so; do
  if [ $lib = default ]; then unset HERO_SIGN_LIB; else export HERO_SIGN_LIB=$PWD/$lib; fi
  echo "== $lib" >> $OUT/sweep.txt
  timeout 600 python tools/variant_sweep.py --sets 128f --count 4096 --reps 5 --tree-split 2 >> $OUT/sweep.txt 2>&1
  timeout 900 python tools/variant_sweep.py --sets 192f,256f --count 16384 --reps 3 --tree-split 2 >> $OUT/sweep.txt 2>&1
done
unset HERO_SIGN_LIB
cat $OUT/sweep.txt
