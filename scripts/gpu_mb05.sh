#!/bin/bash
# Qwen2.5-0.5B shape: micro-batch sweep at ~equal tokens per optimizer step (one B200).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/mb05
for cfg in "16 8" "24 5" "32 4" "16 8" "24 5" "32 4"; do
  set -- $cfg
  timeout 900 python bench.py --micro-batch $1 --grad-accum $2 --steps 4 --warmup 3 --no-cpu-baseline --profile-json gpurun_out/mb05/mb_$1.json > gpurun_out/mb05/mb_$1.log 2>&1
  echo "mb=$1 ga=$2 rc=$?"; python scripts/ab_line.py "0.5B mb=$1" gpurun_out/mb05/mb_$1.json 2>/dev/null
done
