#!/bin/bash
# host-side phases of hs_sign_batch_ex for small batches (trace build): start, after checks, after staging, after run_batch, after drain, end
OUT=gpurun_out/r02bl; mkdir -p $OUT
HERO_SIGN_LIB=paper_2512_23969_b200/libherosign_htrace.so timeout 300 python tools/latency_probe.py --sets 128f --counts 1 --reps 10 > $OUT/probe.txt 2> $OUT/trace.txt
tail -12 $OUT/trace.txt; cut -c1-150 $OUT/probe.txt
