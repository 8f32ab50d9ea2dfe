#!/bin/bash
# Round evidence: launch lists per set, full ncu captures of the dominant kernels (exported to CSV).
OUT=gpurun_out
for s in 128f 192f 256f; do
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$s.csv \
    python tools/ncu_target.py --set $s --count 4096 --runs 2 --mode 0 > $OUT/launches_$s.log 2>&1
done
for spec in "128f tree_sign" "256f tree_sign" "192f fors_sign" "128f tree_shared"; do
  set -- $spec
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -c 1 -o /tmp/ev_$1_$2 -f \
    python tools/ncu_target.py --set $1 --count 4096 --runs 1 --mode 1 > $OUT/ncu_ev_$1_$2.log 2>&1
  ncu -i /tmp/ev_$1_$2.ncu-rep --page raw --csv > $OUT/ev_$1_$2_raw.csv 2>&1
done
ncu -i /tmp/ev_128f_tree_sign.ncu-rep --page source --csv > $OUT/ev_128f_tree_sign_source.csv 2>&1
ncu -i /tmp/ev_128f_tree_sign.ncu-rep --page details --csv > $OUT/ev_128f_tree_sign_details.csv 2>&1
