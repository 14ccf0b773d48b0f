#!/bin/bash
# Optimizer-step batch (gradient accumulation) sweep of the benches on one B200.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ga
for ga in 1 8 31; do
  timeout 900 python bench.py --grad-accum $ga --steps 5 --warmup 3 --no-cpu-baseline --profile-json gpurun_out/ga/ga_$ga.json > gpurun_out/ga/ga_$ga.log 2>&1
  python scripts/ab_line.py "0.5B GA=$ga" gpurun_out/ga/ga_$ga.json
done
for ga in 1 16; do
  timeout 900 python bench.py --config llama-7b --micro-batch 8 --grad-accum $ga --steps 3 --warmup 3 --no-cpu-baseline --profile-json gpurun_out/ga/ga7_$ga.json > gpurun_out/ga/ga7_$ga.log 2>&1
  python scripts/ab_line.py "7B GA=$ga" gpurun_out/ga/ga7_$ga.json
done
