cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/attn_modes.py 2>&1 | tail -4
QTB_ATTN_TC=0 timeout 300 python scripts/attn_modes.py 2>&1 | tail -4
timeout 1200 python -m pytest tests/ -x -q -m gpu --timeout=300 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --profile-json gpurun_out/bench_profile.json > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
python -c "
import json;d=json.load(open('gpurun_out/bench_profile.json'));l=d['line'];print(l['value'],l['ms_per_step'],l['mfu'],l['clocks']);print(json.dumps(l['kernel_classes']))"
