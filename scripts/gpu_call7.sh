cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ncu
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:fwd_tc_kernel -c 1 -o gpurun_out/ncu/attn_fwd_tc python scripts/profile_step.py > gpurun_out/ncu/attn.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/ncu/attn_fwd_tc.ncu-rep --page details --csv > gpurun_out/ncu/attn_fwd_tc.details.csv
ncu -i gpurun_out/ncu/attn_fwd_tc.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu/attn_fwd_tc.source.csv 2>/dev/null
ls -la gpurun_out/ncu/
rm -f gpurun_out/ncu/attn_fwd_tc.ncu-rep
