cd $GRAFT_REPO_ROOT
for b in 16 32 64 100; do echo "budget $b KB"; QTB_RF_SMEM=$b timeout 300 python scripts/elem_bench.py 2>&1 | head -4; done
timeout 300 python scripts/elem_bench.py 2>&1 | tail -4
