#!/bin/bash
# On-device tuning of every set on the final build (narrow FORS_Sign, mx248p4 in the path list).
OUT=gpurun_out/r02ck; mkdir -p $OUT
timeout 2400 python tools/tune_all.py --out $OUT/tuning.json > $OUT/tuning_on_device.txt 2>&1; tail -c 3000 $OUT/tuning_on_device.txt
