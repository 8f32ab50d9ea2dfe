#!/bin/bash
# Small-batch config sweep: tiny FORS layout (one tree per CTA) with all levels in the CTA, native SHA path, one stream.
OUT=gpurun_out/r02u; mkdir -p $OUT
NAT='"variant": {"FORS_Sign": 0, "TREE_Sign": 0, "WOTS_Sign": 0, "host": 0}'
for s in "128f 6" "192f 8" "256f 9"; do set -- $s
  timeout 600 python tools/small_batch_sweep.py --set $1 --counts 1,4,16,64,256 \
    --cfg base='{}' --cfg s1='{"streams": 1}' \
    --cfg tiny0='{"fors_trees_per_set": 1, "fors_sets_fused": 1}' \
    --cfg tinyL="{\"fors_trees_per_set\": 1, \"fors_sets_fused\": 1, \"fors_cta_levels\": $2}" \
    --cfg tinyL_s1="{\"fors_trees_per_set\": 1, \"fors_sets_fused\": 1, \"fors_cta_levels\": $2, \"streams\": 1}" \
    --cfg tinyL_nat="{\"fors_trees_per_set\": 1, \"fors_sets_fused\": 1, \"fors_cta_levels\": $2, $NAT}" \
    >> $OUT/sweep.txt 2>&1
done
cat $OUT/sweep.txt
