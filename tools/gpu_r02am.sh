#!/bin/bash
# verify kernel compiled per SHA path (experiment build, reverted: verify dispatched on the TREE_Sign slot and verify_rate.py --variants): rate per path, 65536 and 16384 signatures.
OUT=gpurun_out/r02am; mkdir -p $OUT
timeout 900 python tools/verify_rate.py --count 65536 --reps 3 --variants 0,1,2,3,4,5 > $OUT/verify_paths.txt 2>&1; cat $OUT/verify_paths.txt
timeout 900 python tools/verify_rate.py --count 16384 --reps 3 --variants 0,2 >> $OUT/verify_paths.txt 2>&1; tail -3 $OUT/verify_paths.txt
