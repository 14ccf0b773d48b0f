#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_deferred_gpu.py -x -q > gpurun_out/defer_t.log 2>&1; echo "defer tests rc=$?"; tail -3 gpurun_out/defer_t.log
for d in 1 0; do
QTB_DEFER_ADAMW=$d timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b05_$d.log 2>&1; echo "b05 defer=$d rc=$?"; tail -1 gpurun_out/b05_$d.log | cut -c1-150
QTB_DEFER_ADAMW=$d timeout 400 python bench.py --config llama-7b --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b7_$d.log 2>&1; echo "b7 defer=$d rc=$?"; tail -1 gpurun_out/b7_$d.log | cut -c1-150
done
