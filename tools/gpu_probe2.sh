#!/bin/bash
# pipe / SHA-path probes with ncu pipe and stall counters (one GPU).
OUT=gpurun_out/probe2; mkdir -p $OUT
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv > $OUT/clocks.txt
./tools/pipe_probe2 > $OUT/pipe_probe2.txt 2>&1
./tools/sha_probe2 > $OUT/sha_probe2.txt 2>&1
M=sm__inst_executed_pipe_alu.sum,sm__inst_executed_pipe_fmaheavy.sum,sm__inst_executed_pipe_fmalite.sum,sm__inst_executed_pipe_fma.sum,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fmalite_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__inst_executed.sum,smsp__warps_eligible.avg.per_cycle_active,smsp__warps_active.avg.per_cycle_active
timeout 600 ncu --clock-control none -k regex:chain --launch-skip 1 --launch-count 1 --section WarpStateStats --section SchedulerStats --metrics $M --csv --page raw ./tools/sha_probe2 Fast > $OUT/ncu_Fast.csv 2>&1
for v in Native 000S1AW 100S1A- 000S2A- 000-1A-; do
  timeout 600 ncu --clock-control none -k regex:chain --launch-skip 1 --launch-count 1 --section WarpStateStats --section SchedulerStats --metrics $M --csv --page raw ./tools/sha_probe2 $v > $OUT/ncu_$v.csv 2>&1
done
