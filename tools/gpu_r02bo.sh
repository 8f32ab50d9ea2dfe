#!/bin/bash
# Randomised GPU-vs-oracle soak (random sets, batches, keys, opt_rand and engine configs), 8 minutes.
OUT=gpurun_out/r02bo; mkdir -p $OUT
timeout 900 python tools/fuzz_gpu.py --minutes 8 --seed 2026 > $OUT/fuzz.txt 2>&1; echo "rc=$?"; tail -5 $OUT/fuzz.txt
