#!/bin/bash
# End-of-round evidence on the final code: suite, smoke, bench + reference arm, launch list of the bench
# command, full ncu capture of the dominant kernel, config-5 stress, compute-sanitizer on smoke.
OUT=gpurun_out/final; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q --durations=10 > $OUT/pytest.txt 2>&1; tail -2 $OUT/pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1; tail -1 $OUT/smoke.txt
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
python - <<'PY'
import json
d=json.loads(open("gpurun_out/final/bench.json").read().strip().splitlines()[-1])
print(d["value"], d["e2e"]["value"], d["roofline"]["frac"], d["launch_latency"]["e2e_small_batch_us"], d["launch_latency"]["device_small_batch_us"], d["clocks"])
for k,o in d["other_sets"].items(): print(k, o["value"], o["e2e"]["value"], o["roofline"]["frac"], o["launch_latency"]["e2e_small_batch_us"], o["launch_latency"]["device_small_batch_us"])
r=json.loads(open("gpurun_out/final/bench_ref.json").read().strip().splitlines()[-1]); print("ref", r["value"])
PY
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_bench_cmd.csv python bench.py --single-set --steps 2 --warmup 1 --no-cpu-baseline --check 2 > $OUT/bench_under_ncu.log 2>&1
python tools/launch_summary.py $OUT/launches_bench_cmd.csv > $OUT/launches_bench_cmd.md 2>&1; head -8 $OUT/launches_bench_cmd.md
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tree_chain -c 1 -o $OUT/tree_chain128f -f python tools/ncu_target.py --set 128f --count 4096 --runs 1 --mode 1 > $OUT/ncu_full.log 2>&1
timeout 2400 python tools/stress_c5.py > $OUT/stress_c5.txt 2>&1; grep '"set"' $OUT/stress_c5.txt
# compute-sanitizer is closed on this GPU pool (runs under it left GPUs needing a reset); the last clean
# memcheck / racecheck / synccheck / initcheck runs are in profiles/sanitizer/ and profiles/r02c_*.
