#!/bin/bash
L=paper_2512_15306_b200/libqtrain_b200.so
timeout 900 python -m pytest tests/test_fused_gpu.py tests/test_parity_more_gpu.py -x -q -k "rms or norm" 2>&1 | tail -2
RMS_M=8192 RMS_D=4096 timeout 300 python scripts/rms_ab.py $L 2>&1 | grep rms_ | sed 's/^/7b /'
RMS_M=4096 RMS_D=5120 timeout 300 python scripts/rms_ab.py $L 2>&1 | grep rms_ | sed 's/^/14b /'
