cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest -q tests/test_bench_shapes_gpu.py tests/test_model_gpu.py tests/test_parity_more_gpu.py --timeout=600 > gpurun_out/t1.log 2>&1; echo "t1 rc=$?"
tail -15 gpurun_out/t1.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench.log | cut -c1-300
python - <<'P'
import json
l=json.loads(open('gpurun_out/bench.log').read().strip().splitlines()[-1])
print(json.dumps(l.get('kernel_classes'), indent=0))
P
