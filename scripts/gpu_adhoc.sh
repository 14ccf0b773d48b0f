#!/bin/bash
mkdir -p gpurun_out
L=paper_2512_15306_b200/libqtrain_b200.so
cp $L /tmp/new.so
cp scratch/old.so $L; timeout 300 python scripts/attn_time.py > gpurun_out/attn_old.log 2>&1; echo "old"; tail -2 gpurun_out/attn_old.log
cp /tmp/new.so $L; timeout 300 python scripts/attn_time.py > gpurun_out/attn_new.log 2>&1; echo "new"; tail -2 gpurun_out/attn_new.log
timeout 600 python -m pytest tests/test_fused_gpu.py tests/test_bench_shapes_gpu.py -x -q -k "attention or attn" > gpurun_out/a1.log 2>&1; echo "attn rc=$?"; tail -3 gpurun_out/a1.log
