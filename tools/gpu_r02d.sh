#!/bin/bash
# FORS launch-bound A/B (768 vs 512 for 192f/256f) + tree_chain pipe counters + full capture with source.
OUT=gpurun_out/r02d; mkdir -p $OUT
timeout 900 python tools/lib_ab.py --libs paper_2512_23969_b200/libherosign_b200.so,paper_2512_23969_b200/libherosign_lb512.so --sets 192f:16384,256f:16384 --rounds 3 > $OUT/lib_ab_lb512.txt 2>&1
M=smsp__inst_executed_pipe_alu.sum,smsp__inst_executed_pipe_fma.sum,smsp__inst_executed_pipe_fmaheavy.sum,smsp__inst_executed_pipe_fmalite.sum,smsp__inst_executed.sum,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active
timeout 600 ncu --metrics $M --clock-control none -k regex:tree_chain -c 1 --csv python tools/ncu_target.py --set 128f --count 1024 --runs 1 --mode 1 > $OUT/chain_pipes.csv 2> $OUT/chain_pipes.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tree_chain -c 1 -o $OUT/tree_chain128f -f python tools/ncu_target.py --set 128f --count 4096 --runs 1 --mode 1 > $OUT/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fors_sign -c 1 -o $OUT/fors256f -f python tools/ncu_target.py --set 256f --count 2048 --runs 1 --mode 1 > $OUT/ncu_fors.log 2>&1
ls -la $OUT
