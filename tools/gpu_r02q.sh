#!/bin/bash
# DRAM traffic of the per-message TREE_Sign kernels per set; full captures of tree_leaf / tree_merkle (128f) and fors_sign (192f).
OUT=gpurun_out/r02q; mkdir -p $OUT
for s in 128f 192f 256f; do
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k 'regex:tree_(chain|leaf|merkle|root)' --csv python tools/ncu_target.py --set $s --count 4096 --runs 1 --mode 1 > $OUT/traffic_$s.csv 2> $OUT/traffic_$s.err
done
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:tree_(leaf|merkle)' -c 2 -o $OUT/tree_leaf_merkle128f -f python tools/ncu_target.py --set 128f --count 4096 --runs 1 --mode 1 > $OUT/ncu1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:fors_(sign|level)' -c 3 -o $OUT/fors192f -f python tools/ncu_target.py --set 192f --count 4096 --runs 1 --mode 1 > $OUT/ncu2.log 2>&1
ls $OUT
