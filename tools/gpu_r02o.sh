#!/bin/bash
# overlap 1 (FORS || TREE streams, concurrent sub-batches) vs 0 (one stream order), device and e2e; T sweep with overlap 0.
OUT=gpurun_out/r02o; mkdir -p $OUT
for s in "128f 4096" "192f 16384" "256f 16384"; do set -- $s
  timeout 900 python tools/ab_config.py --set $1 --count $2 --rounds 3 --e2e --a '{"tree_split": 2, "overlap": true}' --b '{"tree_split": 2, "overlap": false}' >> $OUT/ab_overlap.txt 2>&1
done
cat $OUT/ab_overlap.txt
for s in "192f 16384" "128f 4096"; do set -- $s
  timeout 900 python tools/ab_config.py --set $1 --count $2 --rounds 2 --e2e --a '{"tree_split": 2, "overlap": false, "streams": 2}' --b '{"tree_split": 2, "overlap": false, "streams": 4}' >> $OUT/ab_T.txt 2>&1
done
cat $OUT/ab_T.txt
