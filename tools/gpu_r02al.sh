#!/bin/bash
# verify throughput per SHA path of the verify kernel (0 native, 1 fast, 2.. Mx masks 248,232,104,184).
OUT=gpurun_out/r02al; mkdir -p $OUT
timeout 900 python tools/verify_rate.py --count 65536 --reps 3 --variants 0,1,2,3,4,5 > $OUT/verify_paths.txt 2>&1; cat $OUT/verify_paths.txt
