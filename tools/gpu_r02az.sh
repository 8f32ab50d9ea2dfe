#!/bin/bash
# Source-level captures of fors_sign (192f, 256f) and fors_level / tree_leaf (192f) for SASS execution-count analysis.
OUT=gpurun_out/r02az; mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fors_sign -c 1 -o $OUT/fors192f -f python tools/ncu_target.py --set 192f --count 4096 --runs 1 --mode 1 > $OUT/ncu1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fors_sign -c 1 -o $OUT/fors256f -f python tools/ncu_target.py --set 256f --count 4096 --runs 1 --mode 1 > $OUT/ncu2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fors_level|tree_leaf|shared_chain" -c 3 -o $OUT/misc192f -f python tools/ncu_target.py --set 192f --count 4096 --runs 1 --mode 1 > $OUT/ncu3.log 2>&1
ls -la $OUT
