#!/bin/bash
# tree_root T_len words double-buffered in registers (small graphs): latency A/B vs HEAD, GPU suite.
OUT=gpurun_out/r02bf; mkdir -p $OUT
timeout 900 python tools/lat_ab.py --libs paper_2512_23969_b200/libherosign_old.so,paper_2512_23969_b200/libherosign_b200.so --counts 1,4,16 --rounds 3 > $OUT/lat_ab.txt 2>&1; cat $OUT/lat_ab.txt
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest.txt 2>&1; tail -2 $OUT/pytest.txt
