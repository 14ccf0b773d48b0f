cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_model_gpu.py -q -m gpu -k "graph or train_step or determinism" 2>&1 | tail -2
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b.log 2>&1
python -c "
import json;l=json.loads(open('gpurun_out/b.log').read().strip().splitlines()[-1]);print(round(l['value']), l['ms_per_step'], l['clocks']['sm_mhz'], l['e2e'])"
