# A/B of an env switch on the 0.5B bench: VAR=name bash scripts/gpu_ab.sh
cd $GRAFT_REPO_ROOT
for v in 0 1 0 1; do
  env $VAR=$v timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --profile-json gpurun_out/ab_$v.json > /dev/null 2>&1
  python scripts/ab_line.py "$VAR=$v" gpurun_out/ab_$v.json
done
