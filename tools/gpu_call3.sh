#!/bin/bash
OUT=gpurun_out
mkdir -p $OUT
timeout 600 python -m pytest tests -m gpu -x -q > $OUT/tests3.txt 2>&1
./tools/pipe_probe > $OUT/pipe_probe.txt 2>&1
for v in 0 1; do timeout 120 python tools/ncu_target.py --set 128f --count 4096 --runs 3 --mode 1 --variant $v > $OUT/variant3_$v.txt 2>&1; done
for v in 0 1; do
timeout 600 ncu --section ComputeWorkloadAnalysis --section SchedulerStats --section WarpStateStats --section InstructionStats --metrics sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:tree_sign -c 1 -o /tmp/tree_v$v -f python tools/ncu_target.py --set 128f --count 4096 --runs 1 --mode 1 --variant $v > $OUT/ncu_v$v.log 2>&1
ncu -i /tmp/tree_v$v.ncu-rep --page raw --csv > $OUT/tree_v${v}_raw.csv 2>&1
ncu -i /tmp/tree_v$v.ncu-rep --page details --csv > $OUT/tree_v${v}_details.csv 2>&1
done
du -sh $OUT
