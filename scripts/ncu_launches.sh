set -x
cd $GRAFT_REPO_ROOT
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 1200 -c 1100 --csv --log-file gpurun_out/launches_05b.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
tail -3 gpurun_out/ncu_bench.log
wc -l gpurun_out/launches_05b.csv
