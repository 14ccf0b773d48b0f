cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py --config llama-7b --micro-batch 8 --steps 5 --warmup 3 --no-cpu-baseline --profile-json gpurun_out/bench_7b.json > gpurun_out/bench_7b.log 2>&1; echo "7b rc=$?"
tail -2 gpurun_out/bench_7b.log | cut -c1-1500
timeout 900 python bench.py --config qwen2.5-1.5b --micro-batch 8 --recompute block --steps 5 --warmup 3 --no-cpu-baseline --profile-json gpurun_out/bench_15b.json > gpurun_out/bench_15b.log 2>&1; echo "1.5b rc=$?"
tail -2 gpurun_out/bench_15b.log | cut -c1-1500
