cd $GRAFT_REPO_ROOT
timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/memcheck.log 2>&1; echo "memcheck rc=$?"
tail -15 gpurun_out/memcheck.log
