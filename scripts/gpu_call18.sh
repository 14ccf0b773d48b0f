cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ncu
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:adamw_kernel -c 1 -o gpurun_out/ncu/adamw python scripts/profile_step.py > gpurun_out/ncu/adamw.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/ncu/adamw.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu/adamw.source.csv 2>/dev/null
ncu -i gpurun_out/ncu/adamw.ncu-rep --page details --csv > gpurun_out/ncu/adamw.details.csv 2>/dev/null
rm -f gpurun_out/ncu/adamw.ncu-rep
