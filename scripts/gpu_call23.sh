cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ncu
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:rms_chain_kernel -c 1 -o gpurun_out/ncu/chain7b python scripts/profile_step.py --config llama-7b --micro-batch 8 > gpurun_out/ncu/chain7b.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/ncu/chain7b.ncu-rep --page details --csv > gpurun_out/ncu/chain7b.details.csv
ncu -i gpurun_out/ncu/chain7b.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu/chain7b.source.csv 2>/dev/null
rm -f gpurun_out/ncu/chain7b.ncu-rep
