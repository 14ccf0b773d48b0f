cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/acc
python scripts/gemm_7b.py > gpurun_out/acc/gemm_7b.txt 2>&1; cat gpurun_out/acc/gemm_7b.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel --launch-skip 22 -c 1 -o gpurun_out/acc/wgrad_acc python scripts/gemm_7b.py > /dev/null 2>&1; echo "ncu1 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel --launch-skip 33 -c 1 -o gpurun_out/acc/wgrad_plain python scripts/gemm_7b.py > /dev/null 2>&1; echo "ncu2 rc=$?"
