#!/bin/bash
# Per-set sub-batch head weight (4 / 8 / 8) vs 4 everywhere: public call end to end, interleaved processes.
OUT=gpurun_out/r02ch; mkdir -p $OUT
L=paper_2512_23969_b200/libherosign_b200.so,swlibs/libhs_w4.so
timeout 900 python tools/ab_e2e.py --libs $L --set 192f --count 16384 > $OUT/ab_192f.txt 2>&1
timeout 1200 python tools/ab_e2e.py --libs $L --set 256f --count 65536 > $OUT/ab_256f.txt 2>&1
timeout 600 python tools/ab_e2e.py --libs $L --set 128f --count 4096 > $OUT/ab_128f.txt 2>&1
cat $OUT/ab_*.txt
