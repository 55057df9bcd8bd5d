cd $GRAFT_REPO_ROOT
timeout 1700 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4e.csv python scripts/three_runs.py 2 > gpurun_out/ncu_c4e.log 2>&1
python scripts/launch_summary.py gpurun_out/launches_c4e.csv | head -40
