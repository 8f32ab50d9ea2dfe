#!/bin/bash
# Lone-thread SHA-256 latency probe; full ncu captures (source-level stall sampling) of the 1-message critical-path kernels.
OUT=gpurun_out/r02t; mkdir -p $OUT
timeout 120 tools/lat_probe > $OUT/lat_probe.txt 2>&1; cat $OUT/lat_probe.txt
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:msg_prep|fors_pk|tree_leaf|fors_sign|tree_chain|fors_level' -c 12 -o $OUT/small128f -f python tools/ncu_target.py --set 128f --count 1 --runs 1 --mode 1 > $OUT/ncu.log 2>&1
tail -3 $OUT/ncu.log; ls -la $OUT
