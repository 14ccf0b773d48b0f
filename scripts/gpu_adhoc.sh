cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python scripts/chain_ab.py > gpurun_out/chain_ab.log 2>&1; echo "chain rc=$?"; cat gpurun_out/chain_ab.log
timeout 1200 python scripts/gemm_sweep.py > gpurun_out/gemm_sweep.log 2>&1; echo "sweep rc=$?"
QTB_CHAIN_ROWS=16 timeout 900 python bench.py --config llama-7b --micro-batch 8 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_7b_c16.log 2>&1; echo "7b c16 rc=$?"; tail -1 gpurun_out/bench_7b_c16.log | cut -c1-200
timeout 1500 python -m pytest -q tests/test_model_gpu.py tests/test_fused_gpu.py tests/test_gemm_gpu.py tests/test_optim_gpu.py -x --timeout=600 > gpurun_out/t5.log 2>&1; echo "t5 rc=$?"; tail -3 gpurun_out/t5.log
