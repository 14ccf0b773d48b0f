cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/fin
timeout 2400 python -m pytest tests/ -q -m gpu --timeout=900 > gpurun_out/fin/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/fin/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/fin/smoke.log
timeout 900 python bench.py > gpurun_out/fin/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/fin/bench.log | cut -c1-250
