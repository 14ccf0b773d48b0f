cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/attn_fwd2q.py > gpurun_out/fwd2q.log 2>&1; echo "fwd2q rc=$?"; cat gpurun_out/fwd2q.log | tail -20
