cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py --config llama-7b --micro-batch 8 --steps 5 --warmup 3 --no-cpu-baseline --profile-json gpurun_out/bench_7b.json > gpurun_out/bench_7b.log 2>&1; echo "7b rc=$?"
python -c "
import json;d=json.load(open('gpurun_out/bench_7b.json'));l=d['line'];print(l['value'],l['ms_per_step'],l['mfu'],l['clocks']);print(json.dumps(l['kernel_classes']))"
timeout 900 python bench.py --config qwen2.5-1.5b --micro-batch 8 --recompute block --steps 5 --warmup 3 --no-cpu-baseline --profile-json gpurun_out/bench_15b.json > gpurun_out/bench_15b.log 2>&1; echo "1.5b rc=$?"
python -c "
import json;d=json.load(open('gpurun_out/bench_15b.json'));l=d['line'];print(l['value'],l['ms_per_step'],l['mfu'],l['clocks']);print(json.dumps(l['kernel_classes']))"
