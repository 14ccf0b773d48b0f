cd $GRAFT_REPO_ROOT
timeout 300 python scripts/elem_bench.py 2>&1 | tail -12
timeout 1200 python -m pytest tests/test_fused_gpu.py tests/test_quant_gpu.py tests/test_model_gpu.py -x -q -m gpu --timeout=300 2>&1 | tail -3
