cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/ -q -m gpu --timeout=600 > gpurun_out/pt.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pt.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --profile-json gpurun_out/bench_profile.json > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
python scripts/ab_line.py head gpurun_out/bench_profile.json
python -c "import json;d=json.load(open('gpurun_out/bench_profile.json'));print(d['line']['kernel_classes']['quant'], d['line']['gpu_launches_per_step'])"
