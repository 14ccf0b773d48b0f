cd $GRAFT_REPO_ROOT
timeout 1200 ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/traffic_05b.csv python scripts/profile_step.py > gpurun_out/ncu_traffic.log 2>&1; echo "ncu rc=$?"
python scripts/traffic_summary.py gpurun_out/traffic_05b.csv gpurun_out/traffic_05b.json
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python scripts/profile_step.py > gpurun_out/ncu_launch.log 2>&1; echo "ncu rc=$?"
python scripts/summarize_launches.py gpurun_out/launches.csv 60 > gpurun_out/launches_summary.txt; head -30 gpurun_out/launches_summary.txt
