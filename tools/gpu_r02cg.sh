#!/bin/bash
# Randomised GPU-vs-oracle soak on the current path list (mx248p4 compiled in, 256f FORS_Sign on it).
OUT=gpurun_out/r02cg; mkdir -p $OUT
timeout 900 python tools/fuzz_gpu.py --minutes 10 --seed 4242 > $OUT/fuzz_gpu.txt 2>&1; tail -2 $OUT/fuzz_gpu.txt
