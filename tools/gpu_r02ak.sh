#!/bin/bash
# ncu full capture of the GPU verification kernel (128f, 65536 signatures).
OUT=gpurun_out/r02ak; mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:verify_thread -c 1 -o $OUT/verify128f -f python tools/ncu_verify.py > $OUT/ncu.log 2>&1
tail -2 $OUT/ncu.log
python tools/ncu_summary.py $OUT/verify128f.ncu-rep 2>&1 | head -40
