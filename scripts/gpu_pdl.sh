#!/bin/bash
# PDL (programmatic dependent launch) evidence on one B200: per-boundary gap
# microbenchmark, parity tests with PDL on, and QTB_PDL=0/1 A/B of the benches.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/pdl
nvcc -gencode arch=compute_100a,code=sm_100a -O3 scripts/micro/pdl_gap.cu -o /tmp/pdl_gap && timeout 120 /tmp/pdl_gap > gpurun_out/pdl/gap.txt 2>&1
cat gpurun_out/pdl/gap.txt
timeout 900 python -m pytest tests/test_model_gpu.py tests/test_gemm_gpu.py -q -m gpu -x --timeout=600 > gpurun_out/pdl/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pdl/pytest.log
for v in 0 1 0 1; do
  QTB_PDL=$v timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --profile-json gpurun_out/pdl/ab_$v.json > /dev/null 2>&1
  python scripts/ab_line.py "QTB_PDL=$v" gpurun_out/pdl/ab_$v.json
done
for v in 0 1; do
  QTB_PDL=$v timeout 600 python bench.py --config llama-7b --micro-batch 8 --steps 5 --warmup 3 --no-cpu-baseline --profile-json gpurun_out/pdl/ab7_$v.json > /dev/null 2>&1
  python scripts/ab_line.py "7B QTB_PDL=$v" gpurun_out/pdl/ab7_$v.json
done
