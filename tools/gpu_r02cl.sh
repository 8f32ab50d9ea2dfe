#!/bin/bash
# ncu full capture of FORS_Sign (256f, narrow kernel, 4 fused sets) and (192f, narrow kernel) on the final build.
OUT=gpurun_out/r02cl; mkdir -p $OUT
python tools/ncu_target.py --set 256f --count 2048 --runs 1 --mode 1 > $OUT/plain256.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fors_sign -c 1 -o $OUT/fors256f -f python tools/ncu_target.py --set 256f --count 2048 --runs 1 --mode 1 > $OUT/ncu256.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fors_sign -c 1 -o $OUT/fors192f -f python tools/ncu_target.py --set 192f --count 2048 --runs 1 --mode 1 > $OUT/ncu192.log 2>&1
tail -2 $OUT/ncu256.log $OUT/ncu192.log
