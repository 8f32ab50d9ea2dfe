#!/bin/bash
# usage: tools/gpu.sh <name> '<command run on the box from the repo root>' [timeout_s]
# Runs one gpurun call in the background; log in gpurun_out/<name>.log
cd /root/repo || exit 1
name=$1; cmd=$2; t=${3:-1500}
( timeout $((t + 1200)) /usr/local/graft/bin/gpurun --timeout "$t" -- "$cmd" > "gpurun_out/$name.log" 2>&1
  echo "EXIT $?" >> "gpurun_out/$name.log" ) &
