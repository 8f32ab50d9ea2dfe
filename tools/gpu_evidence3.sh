#!/bin/bash
# Final round-1 evidence for the current code: bench (+ reference arm), launch
# lists per set (graph mode), full ncu captures of the kernels on the path,
# BASELINE config 5 stress.
OUT=${EVOUT:-gpurun_out/ev3}; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 900 python bench.py --impl reference > $OUT/ref.json 2> $OUT/ref.err
for s in 128f 192f 256f; do
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$s.csv \
    python tools/ncu_target.py --set $s --count 4096 --runs 2 --mode 0 > $OUT/launches_$s.log 2>&1
done
for spec in "128f tree_chain 0" "192f tree_chain 0" "256f tree_chain 0" "128f tree_root 0" "192f fors_sign 0" \
            "192f fors_level 3" "256f fors_sign 0" "128f shared_chain 0"; do
  set -- $spec
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 --launch-skip $3 -c 1 -o /tmp/ev_$1_$2 -f \
    python tools/ncu_target.py --set $1 --count 4096 --runs 1 --mode 1 > $OUT/ncu_$1_$2.log 2>&1
  ncu -i /tmp/ev_$1_$2.ncu-rep --page raw --csv > $OUT/raw_$1_$2.csv 2>&1
done
ncu -i /tmp/ev_128f_tree_chain.ncu-rep --page source --csv > $OUT/src_128f_tree_chain.csv 2>&1
timeout 1500 python tools/stress_c5.py > $OUT/stress_c5.txt 2>&1
