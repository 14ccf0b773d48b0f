cd $GRAFT_REPO_ROOT
timeout 300 python scripts/elem_bench.py 2>&1 | head -4
timeout 1200 python -m pytest tests/test_fused_gpu.py tests/test_model_gpu.py -x -q -m gpu --timeout=300 2>&1 | tail -2
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_7b.csv python scripts/profile_step.py --config llama-7b --micro-batch 8 > gpurun_out/ncu_launch.log 2>&1; echo "ncu rc=$?"
python scripts/summarize_launches.py gpurun_out/launches_7b.csv 40 | grep -E "total|rms|colsum"
