cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for r in 32 16; do
QTB_CHAIN_ROWS=$r timeout 900 python -m pytest -q tests/test_fused_gpu.py -k rmsnorm --timeout=600 > gpurun_out/rms_$r.log 2>&1; echo "rows=$r rc=$?"; tail -3 gpurun_out/rms_$r.log
done
