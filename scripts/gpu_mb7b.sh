#!/bin/bash
# Llama-7B shape: micro-batch sweep at a fixed accumulation depth (one B200).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/mb
for mb in 8 12 16; do
  timeout 900 python bench.py --config llama-7b --micro-batch $mb --grad-accum 8 --steps 2 --warmup 3 --no-cpu-baseline --profile-json gpurun_out/mb/mb_$mb.json > gpurun_out/mb/mb_$mb.log 2>&1
  echo "mb=$mb rc=$?"; python scripts/ab_line.py "7B mb=$mb" gpurun_out/mb/mb_$mb.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/mb/mb_$mb.json'))['line'];print(d['mfu'],d['device_bytes']/1e9)" 2>/dev/null
  tail -2 gpurun_out/mb/mb_$mb.log | cut -c1-300
done
