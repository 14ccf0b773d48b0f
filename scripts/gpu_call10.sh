cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ncu
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rms_fwd_fused -s 2 -c 1 -o gpurun_out/ncu/rmsf python scripts/elem_bench.py > gpurun_out/ncu/rmsf.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/ncu/rmsf.ncu-rep --page details --csv > gpurun_out/ncu/rmsf.details.csv
ncu -i gpurun_out/ncu/rmsf.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu/rmsf.source.csv 2>/dev/null
rm -f gpurun_out/ncu/rmsf.ncu-rep
