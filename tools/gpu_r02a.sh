#!/bin/bash
# Round-2 first GPU call: state check, per-pipe instruction counts of the
# TREE_Sign chain kernel, FORS_Sign 256f full capture with source, bench.
OUT=gpurun_out/r02a; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi.txt
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1
M=smsp__inst_executed.sum,smsp__inst_executed_pipe_alu.sum,smsp__inst_executed_pipe_fma.sum,smsp__inst_executed_pipe_fmaheavy.sum,smsp__inst_executed_pipe_fmalite.sum,smsp__inst_executed_pipe_fma_type_fp16.sum,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum
timeout 600 ncu --metrics $M --clock-control none -k regex:tree_chain -c 1 --csv python tools/ncu_target.py --set 128f --count 4096 --runs 1 --mode 1 > $OUT/pipes_tree_chain_128f.csv 2> $OUT/pipes.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fors_sign -c 1 -o $OUT/fors256 -f \
    python tools/ncu_target.py --set 256f --count 4096 --runs 1 --mode 1 > $OUT/ncu_fors256.log 2>&1
ncu -i $OUT/fors256.ncu-rep --page raw --csv > $OUT/raw_fors256.csv 2>&1
ncu -i $OUT/fors256.ncu-rep --page source --csv > $OUT/src_fors256.csv 2>&1
rm -f $OUT/fors256.ncu-rep
timeout 600 python bench.py --single-set --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err
ls -la $OUT
