cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ncu
for k in dq_tc_kernel dkdv_tc_kernel; do
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:$k -c 1 -o gpurun_out/ncu/$k python scripts/profile_step.py > /dev/null 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/ncu/$k.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu/$k.source.csv 2>/dev/null
rm -f gpurun_out/ncu/$k.ncu-rep
done
