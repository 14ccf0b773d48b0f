# Round-end evidence: GPU tests, smoke, default bench line, reference arm, 7B and 1.5B lines,
# one-step launch list + DRAM traffic of the 0.5B step.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ev
timeout 1500 python -m pytest tests/ -q -m gpu --timeout=600 > gpurun_out/ev/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/ev/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/ev/smoke.log
timeout 900 python bench.py > gpurun_out/ev/bench_0.5b.log 2>&1; echo "bench rc=$?"
timeout 900 python bench.py --config llama-7b --micro-batch 8 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ev/bench_7b.log 2>&1; echo "7b rc=$?"
timeout 900 python bench.py --config qwen2.5-1.5b --micro-batch 8 --recompute block --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ev/bench_15b.log 2>&1; echo "1.5b rc=$?"
timeout 1500 python bench.py --config qwen2.5-14b --micro-batch 4 --moments bf16_sr --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ev/bench_14b.log 2>&1; echo "14b rc=$?"
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev/launches_0.5b.csv python scripts/profile_step.py > /dev/null 2>&1; echo "ncu rc=$?"
python scripts/summarize_launches.py gpurun_out/ev/launches_0.5b.csv 60 > gpurun_out/ev/launches_0.5b.txt
timeout 1200 ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev/traffic_0.5b.csv python scripts/profile_step.py > /dev/null 2>&1; echo "traffic rc=$?"
python scripts/traffic_summary.py gpurun_out/ev/traffic_0.5b.csv gpurun_out/ev/traffic_0.5b.json
rm -f gpurun_out/ev/traffic_0.5b.csv
for f in bench_0.5b bench_7b bench_15b bench_14b; do tail -1 gpurun_out/ev/$f.log | cut -c1-300; done
