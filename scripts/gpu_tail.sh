#!/bin/bash
# Tail-split GEMM: kernel check, GEMM / model parity tests, QTB_GEMM_TAIL A/B of the 0.5B bench.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/tail
python scripts/gemm_tail.py > gpurun_out/tail/tail.txt 2>&1; cat gpurun_out/tail/tail.txt
timeout 1200 python -m pytest tests/test_gemm_gpu.py tests/test_bench_shapes_gpu.py tests/test_model_gpu.py tests/test_optim_gpu.py -q -m gpu -x --timeout=900 > gpurun_out/tail/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/tail/pytest.log
for v in 0 1 0 1; do
  QTB_GEMM_TAIL=$v timeout 600 python bench.py --grad-accum 8 --steps 4 --warmup 3 --no-cpu-baseline --profile-json gpurun_out/tail/ab_$v.json > /dev/null 2>&1
  python scripts/ab_line.py "QTB_GEMM_TAIL=$v" gpurun_out/tail/ab_$v.json
done
