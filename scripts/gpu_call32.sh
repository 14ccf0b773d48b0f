cd $GRAFT_REPO_ROOT
for v in 16 4; do
QTB_RF_MIN_ROWS=$v timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l7_$v.csv python scripts/profile_step.py --config llama-7b --micro-batch 8 > /dev/null 2>&1
echo "min_rows=$v"; python scripts/summarize_launches.py gpurun_out/l7_$v.csv 80 | grep -E "total|rms|colsum"
done
