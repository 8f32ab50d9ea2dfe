#!/bin/bash
# Narrow FORS_Sign instantiation (64 registers; 192f <= 256 lanes, 256f <= 512 lanes) vs wide only
# (HS_FORS_NARROW=0): serialised kernel times and graph batch time, libs interleaved in separate
# processes; then the 256f fused-set count on the new lib; then the suite.
OUT=gpurun_out/r02ci; mkdir -p $OUT
timeout 1200 python tools/lib_ab.py --libs paper_2512_23969_b200/libherosign_b200.so,swlibs/libhs_wide.so \
  --sets 192f:16384,256f:16384 --rounds 3 --reps 5 > $OUT/lib_ab.txt 2>&1; cat $OUT/lib_ab.txt | cut -c1-400
timeout 900 python tools/ab_config.py --set 256f --count 16384 --serial --a '{"fors_sets_fused": 7}' --b '{"fors_sets_fused": 4}' > $OUT/ab_fused256.txt 2>&1; cut -c1-300 $OUT/ab_fused256.txt
timeout 600 python tools/ab_config.py --set 192f --count 16384 --serial --a '{"fors_sets_fused": 11}' --b '{"fors_sets_fused": 8}' > $OUT/ab_fused192.txt 2>&1; cut -c1-300 $OUT/ab_fused192.txt
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest.txt 2>&1; tail -2 $OUT/pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1; tail -1 $OUT/smoke.txt
