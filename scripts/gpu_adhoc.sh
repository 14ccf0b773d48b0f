#!/bin/bash
mkdir -p gpurun_out
timeout 300 python scripts/attn_fwd2q.py > gpurun_out/fwd2q.log 2>&1; echo "fwd2q rc=$?"; cat gpurun_out/fwd2q.log | tail -12
timeout 600 python -m pytest tests/test_fused_gpu.py -x -q -k "attention" > gpurun_out/a1.log 2>&1; echo "attn rc=$?"; tail -3 gpurun_out/a1.log
