#!/bin/bash
# C-form rotations (hoistable) vs inline-PTX funnel shifts: GPU suite on the new build, interleaved A/B, SHA-path sweep.
OUT=gpurun_out/r02e; mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest.txt 2>&1
tail -2 $OUT/pytest.txt
timeout 1200 python tools/lib_ab.py --libs paper_2512_23969_b200/libherosign_rotasm.so,paper_2512_23969_b200/libherosign_b200.so --sets 128f:4096,192f:16384,256f:16384 --rounds 3 > $OUT/lib_ab_rotc.txt 2>&1
cat $OUT/lib_ab_rotc.txt
timeout 900 python tools/variant_sweep.py --count 4096 --reps 5 > $OUT/variant_sweep.txt 2>&1
cat $OUT/variant_sweep.txt
