cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python scripts/lm_precision.py 2048 > gpurun_out/lm_precision.log 2>&1; echo "lmprec rc=$?"
timeout 900 python -m pytest -q -x tests/test_parity_more_gpu.py -k width -s > gpurun_out/width.log 2>&1; echo "width rc=$?"
tail -5 gpurun_out/width.log
cat gpurun_out/lm_precision.log
