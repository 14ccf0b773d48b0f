cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/ -q -m gpu -x --timeout=600 2>&1 | tail -2
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l5.csv python scripts/profile_step.py > /dev/null 2>&1
python scripts/summarize_launches.py gpurun_out/l5.csv 40 | grep -E "total|bwd_dot|gemm<0, 0, 0"
