# Launch list (per-kernel durations) of one 0.5B training step, after warm-up.
cd $GRAFT_REPO_ROOT
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 3700 -c 1229 --csv --log-file gpurun_out/launches_05b.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
python scripts/summarize_launches.py gpurun_out/launches_05b.csv 45
