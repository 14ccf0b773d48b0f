# ncu --set full captures of the hot kernels of ONE 0.5B training step (after warm-up),
# via scripts/profile_step.py (cudaProfilerStart/Stop around the step).  Reports are
# reduced to CSV (details page + raw key metrics) on the box; .ncu-rep files are deleted
# unless KEEP_REP=1 (gpurun copies back at most 64 MiB).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ncu
TAG=${TAG:-r01}
EXTRA=${EXTRA:-}
RAWM="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,launch__grid_size,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active"
reduce() {
  ncu -i $1.ncu-rep --page details --csv > $1.details.csv 2>/dev/null
  ncu -i $1.ncu-rep --page raw --csv --metrics $RAWM > $1.raw.csv 2>/dev/null
  [ "${KEEP_REP:-0}" = "1" ] || rm -f $1.ncu-rep
}
if [ -z "${SKIP_GEMM:-}" ]; then
timeout 1200 ncu --profile-from-start off --set full --clock-control none --import-source on \
   -k regex:gemm_kernel -s ${GEMM_SKIP:-92} -c ${GEMM_COUNT:-15} -o gpurun_out/ncu/${TAG}_gemms python scripts/profile_step.py $EXTRA > gpurun_out/ncu/${TAG}_gemms.log 2>&1
echo "gemms rc=$?"; reduce gpurun_out/ncu/${TAG}_gemms
fi
K=${KERNELS:-"adamw_kernel ce_softmax_kernel fwd1_tc_kernel swiglu_bwd_kernel swiglu_fwd_kernel rms_fwd_fused_kernel rms_bwd_fused_kernel quantize_bf16_kernel dq_tc_kernel dkdv_tc_kernel rope_kernel"}
for k in $K; do
  timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on \
     -k regex:"$k" -c 1 -o gpurun_out/ncu/${TAG}_$k python scripts/profile_step.py $EXTRA > gpurun_out/ncu/${TAG}_$k.log 2>&1
  echo "$k rc=$?"; reduce gpurun_out/ncu/${TAG}_$k
done
du -sh gpurun_out/ncu
