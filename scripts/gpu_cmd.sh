cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gemm_gpu.py tests/test_fused_gpu.py -x -q --timeout=60 --timeout-method=thread 2>&1 | tail -3
timeout 300 python scripts/gemm_bench.py 2>&1 | tail -20
timeout 120 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"tc_kernel" -c 3 --csv python scripts/attn_big.py 2>/dev/null | grep -E "kernel" | awk -F'","' '{print $5, $NF}' | cut -c1-40,130-
