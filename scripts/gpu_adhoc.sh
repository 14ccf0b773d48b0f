cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest -q -x tests/test_peer_group_gpu.py tests/test_trainer_gpu.py --timeout=900 > gpurun_out/t2.log 2>&1; echo "t2 rc=$?"
tail -5 gpurun_out/t2.log
timeout 1200 python -m pytest -q tests/test_model_gpu.py tests/test_optim_gpu.py tests/test_parity_more_gpu.py tests/test_cpp_gpu.py "tests/test_bench_shapes_gpu.py::test_cross_entropy_production_path_real_vocab" --timeout=600 > gpurun_out/t3.log 2>&1; echo "t3 rc=$?"
tail -5 gpurun_out/t3.log
