cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_fused_gpu.py tests/test_model_gpu.py -x -q -m gpu --timeout=300 2>&1 | tail -2
timeout 900 python bench.py --config llama-7b --micro-batch 8 --steps 5 --warmup 3 --no-cpu-baseline --profile-json gpurun_out/bench_7b.json > gpurun_out/bench_7b.log 2>&1; echo "7b rc=$?"
python -c "
import json;d=json.load(open('gpurun_out/bench_7b.json'));l=d['line'];print(l['value'],l['ms_per_step'],l['mfu'],l['clocks']);print(json.dumps(l['kernel_classes']))"
