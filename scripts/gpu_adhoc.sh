cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest -q tests/test_offload_gpu.py tests/test_trainer_gpu.py --timeout=600 > gpurun_out/t4.log 2>&1; echo "offload+trainer rc=$?"; tail -3 gpurun_out/t4.log
QTB_LM_TX=0 timeout 600 python -m pytest -q tests/test_parity_more_gpu.py -k llama7b_width -s --timeout=600 > gpurun_out/w0.log 2>&1; echo "lmtx0 rc=$?"; grep -E "passed|failed|Error:" gpurun_out/w0.log | head -5
timeout 600 python -m pytest -q tests/test_parity_more_gpu.py -k qwen05b_width -s --timeout=600 > gpurun_out/w1.log 2>&1; echo "qwen rc=$?"; grep -E "passed|failed|\{" gpurun_out/w1.log | head -5
