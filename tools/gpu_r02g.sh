#!/bin/bash
# BASELINE config 5 stress on the current build (e2e vs device-timed rate at the same mixed-key config).
OUT=gpurun_out/r02g; mkdir -p $OUT
timeout 1500 python tools/stress_c5.py > $OUT/stress_c5.txt 2>&1
cat $OUT/stress_c5.txt
