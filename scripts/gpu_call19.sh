cd $GRAFT_REPO_ROOT
timeout 300 python scripts/attn_modes.py 2>&1 | tail -1
QTB_ATTN_FWD2=1 timeout 300 python scripts/attn_modes.py 2>&1 | tail -1
timeout 1200 python -m pytest tests/ -x -q -m gpu --timeout=300 > gpurun_out/pt.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pt.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --profile-json gpurun_out/bench_profile.json > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
python -c "
import json;d=json.load(open('gpurun_out/bench_profile.json'));l=d['line'];print(l['value'],l['ms_per_step'],l['mfu'],l['clocks']);print(json.dumps(l['kernel_classes']))"
