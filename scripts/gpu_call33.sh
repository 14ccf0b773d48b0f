cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_optim_gpu.py tests/test_model_gpu.py -q -m gpu 2>&1 | tail -1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l5.csv python scripts/profile_step.py > /dev/null 2>&1
python scripts/summarize_launches.py gpurun_out/l5.csv 60 | grep -E "total|adamw|norm_partials|dq_tc|dkdv_tc"
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l7.csv python scripts/profile_step.py --config llama-7b --micro-batch 8 > /dev/null 2>&1
python scripts/summarize_launches.py gpurun_out/l7.csv 60 | grep -E "total|adamw|norm_partials|dq_tc|dkdv_tc"
