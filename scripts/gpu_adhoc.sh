cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench05.log 2>&1; echo "0.5b rc=$?"
python -c "import json;l=json.loads(open('gpurun_out/bench05.log').read().strip().splitlines()[-1]);print(l['value'],l['ms_per_step'],l['clocks']['sm_mhz'],l['mfu'])"
timeout 900 python bench.py --config llama-7b --micro-batch 8 --steps 5 --warmup 3 --no-cpu-baseline --profile-json gpurun_out/prof7b.json > gpurun_out/bench_7b.log 2>&1; echo "7b rc=$?"
python -c "import json;l=json.loads(open('gpurun_out/bench_7b.log').read().strip().splitlines()[-1]);print(l['value'],l['ms_per_step'],l['clocks']['sm_mhz'],l['mfu'])"
timeout 2400 python -m pytest -q tests/test_model_gpu.py tests/test_peer_group_gpu.py tests/test_offload_gpu.py tests/test_trainer_gpu.py tests/test_optim_gpu.py tests/test_cpp_gpu.py --timeout=900 > gpurun_out/t6.log 2>&1; echo "t6 rc=$?"; tail -4 gpurun_out/t6.log
