#!/bin/bash
# First-call cost: lazy vs eager module loading, old vs current library (128f, 65,536-message calls).
OUT=gpurun_out/r02aq; mkdir -p $OUT
for ml in LAZY EAGER; do
  CUDA_MODULE_LOADING=$ml HERO_SIGN_LIB=paper_2512_23969_b200/libherosign_old.so HERO_SIGN_CONFIG=paper_2512_23969_b200/old_tuned.json timeout 600 python tools/e2e_calls.py --calls 3 > $OUT/old_$ml.txt 2>&1
  CUDA_MODULE_LOADING=$ml timeout 600 python tools/e2e_calls.py --calls 3 > $OUT/new_$ml.txt 2>&1
  echo "$ml old $(cat $OUT/old_$ml.txt)"; echo "$ml new $(cat $OUT/new_$ml.txt)"
done
python - <<'PY'
import time, sys
sys.path.insert(0, '.')
t0 = time.perf_counter()
import paper_2512_23969_b200 as hs
eng = hs.get_engine(0)
print("engine open s", round(time.perf_counter() - t0, 3))
PY
