cd $GRAFT_REPO_ROOT
for k in bwd_dkdv_kernel bwd_dq_kernel fwd_kernel; do
timeout 300 ncu --set full --clock-control none --import-source on -k "regex:${k}" -s 12 -c 1 -o gpurun_out/attn_${k} python scripts/attn_modes.py > /dev/null 2>&1
echo $k $?
done
