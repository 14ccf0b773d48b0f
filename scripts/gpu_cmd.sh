cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/ -x -q -m gpu --timeout=120 --timeout-method=thread 2>&1 | tail -5
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['mfu']); print(json.dumps(d['kernel_classes']))"
bash scripts/ncu_launches.sh 2>&1 | head -40
