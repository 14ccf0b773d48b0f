cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_fused_gpu.py -q -m gpu -k rmsnorm 2>&1 | tail -2
for v in 0 1; do
QTB_CHAIN_DIRECT=$v timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l7_$v.csv python scripts/profile_step.py --config llama-7b --micro-batch 8 > /dev/null 2>&1
echo "direct=$v"; python scripts/summarize_launches.py gpurun_out/l7_$v.csv 60 | grep -E "total|rms_chain"
done
