#!/bin/bash
# Config-5 stress on the current code with one untimed warm-up chunk.
OUT=gpurun_out/r02as; mkdir -p $OUT
timeout 2400 python tools/stress_c5.py > $OUT/stress_c5.txt 2>&1; tail -4 $OUT/stress_c5.txt
