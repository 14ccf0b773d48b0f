#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"fwd2q|dkdv|dq_tc" --launch-skip 3 -c 3 -o gpurun_out/attn05 -f python scripts/attn_prof.py 0.5b > gpurun_out/ncu_attn.log 2>&1; echo "ncu rc=$?"; tail -5 gpurun_out/ncu_attn.log
