# Round-end evidence: GPU tests, smoke, default bench line, reference arm, 7B / 1.5B / 14B lines,
# one-step launch lists (0.5B, 7B) + DRAM traffic of the 0.5B step, ncu --set full of the hot kernels.
cd $GRAFT_REPO_ROOT
TAG=${TAG:-r02}
mkdir -p gpurun_out/ev
if [ -z "${SKIP_TESTS:-}" ]; then
timeout 2400 python -m pytest tests/ -q -m gpu --timeout=900 > gpurun_out/ev/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/ev/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/ev/smoke.log
fi
if [ -z "${SKIP_BENCH:-}" ]; then
timeout 900 python bench.py > gpurun_out/ev/bench_0.5b.log 2>&1; echo "bench rc=$?"
timeout 900 python bench.py --grad-accum 1 --no-cpu-baseline > gpurun_out/ev/bench_0.5b_ga1.log 2>&1; echo "bench ga1 rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/ev/bench_reference.log 2>&1; echo "ref rc=$?"
timeout 900 python bench.py --config llama-7b --micro-batch 12 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ev/bench_7b.log 2>&1; echo "7b rc=$?"
timeout 900 python bench.py --config llama-7b --micro-batch 8 --grad-accum 1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ev/bench_7b_ga1.log 2>&1; echo "7b ga1 rc=$?"
timeout 900 python bench.py --config qwen2.5-1.5b --micro-batch 8 --recompute block --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ev/bench_15b.log 2>&1; echo "1.5b rc=$?"
timeout 1500 python bench.py --config qwen2.5-14b --micro-batch 4 --grad-accum 16 --moments bf16_sr --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ev/bench_14b.log 2>&1; echo "14b rc=$?"
fi
if [ -z "${SKIP_NCU:-}" ]; then
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev/launches_0.5b.csv python scripts/profile_step.py --ga 2 > /dev/null 2>&1; echo "ncu rc=$?"
python scripts/summarize_launches.py gpurun_out/ev/launches_0.5b.csv 60 > gpurun_out/ev/launches_0.5b.txt
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev/launches_7b.csv python scripts/profile_step.py --config llama-7b --micro-batch 8 --ga 2 > /dev/null 2>&1; echo "ncu7b rc=$?"
python scripts/summarize_launches.py gpurun_out/ev/launches_7b.csv 60 > gpurun_out/ev/launches_7b.txt
timeout 1200 ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev/traffic_0.5b.csv python scripts/profile_step.py > /dev/null 2>&1; echo "traffic rc=$?"
python scripts/traffic_summary.py gpurun_out/ev/traffic_0.5b.csv gpurun_out/ev/traffic_0.5b.json
rm -f gpurun_out/ev/traffic_0.5b.csv
fi
if [ -z "${SKIP_FULL:-}" ]; then
TAG=${TAG}final KERNELS="adamw_kernel ce_softmax_stats_kernel fwd2q_tc_kernel swiglu_bwd_kernel swiglu_fwd_kernel rms_chain2_kernel rms_bwd_rows_kernel rms_fwd_rows_kernel quantize_bf16_kernel dq_tc_kernel dkdv_tc_kernel rope_kernel" bash scripts/ncu_step.sh
python scripts/ncu_summary.py gpurun_out/ncu/${TAG}final_*.raw.csv > gpurun_out/ncu/${TAG}final_ncu_summary.txt 2>&1
fi
for f in bench_0.5b bench_0.5b_ga1 bench_reference bench_7b bench_7b_ga1 bench_15b bench_14b; do tail -1 gpurun_out/ev/$f.log 2>/dev/null | cut -c1-300; done
