# one ncu --set full capture per kernel of interest (1 GPU, short command)
cd $GRAFT_REPO_ROOT
for k in "rmsnorm_bwd_kernel" "rmsnorm_fwd_kernel" "bwd_dkdv_kernel" "fwd_kernel" "adamw_kernel" "gemm_kernel<0, false, false, 256, 0>"; do
  tag=$(echo "$k" | tr -cd 'a-z_0-9')
  timeout 300 ncu --set full --clock-control none --import-source on -k "regex:${k}" -s 2 -c 1 -o gpurun_out/full_${tag} \
     python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_${tag}.log 2>&1
  echo "$k rc=$?"
done
ls -la gpurun_out/*.ncu-rep
