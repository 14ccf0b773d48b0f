cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest -q -x tests/test_offload_gpu.py --timeout=600 > gpurun_out/t4.log 2>&1; echo "offload rc=$?"; tail -3 gpurun_out/t4.log
timeout 900 python -m pytest -q tests/test_trainer_gpu.py tests/test_cpp_gpu.py --timeout=600 > gpurun_out/t2.log 2>&1; echo "trainer rc=$?"; tail -3 gpurun_out/t2.log
timeout 900 python scripts/attn_plo.py > gpurun_out/attn_plo.log 2>&1; echo "plo rc=$?"; cat gpurun_out/attn_plo.log
timeout 1200 python -m pytest -q tests/test_parity_more_gpu.py tests/test_model_gpu.py --timeout=600 > gpurun_out/t3.log 2>&1; echo "t3 rc=$?"; tail -4 gpurun_out/t3.log
