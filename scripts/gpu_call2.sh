cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/attn_modes.py > gpurun_out/attn_modes.log 2>&1; echo "modes rc=$?"; cat gpurun_out/attn_modes.log | tail -8
QTB_ATTN_TC=1 timeout 300 python scripts/attn_modes.py > gpurun_out/attn_modes_tc.log 2>&1; echo "modes tc rc=$?"; cat gpurun_out/attn_modes_tc.log | tail -8
bash scripts/ncu_step.sh
