cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -q -m gpu --timeout=300 --timeout-method=thread > gpurun_out/pytest_head.log 2>&1; echo "head rc=$?"
tail -25 gpurun_out/pytest_head.log
cd prev_wt
timeout 900 python -m pytest tests/ -q -m gpu --timeout=300 --timeout-method=thread > ../gpurun_out/pytest_prev.log 2>&1; echo "prev rc=$?"
tail -15 ../gpurun_out/pytest_prev.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > ../gpurun_out/bench_prev.log 2>&1; echo "bench rc=$?"
tail -1 ../gpurun_out/bench_prev.log | cut -c1-1500
