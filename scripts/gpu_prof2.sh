cd $GRAFT_REPO_ROOT
timeout 300 python scripts/one_factorize.py c4 > gpurun_out/plain_c4.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python scripts/one_factorize.py c4 > gpurun_out/ncu_c4.log 2>&1
tail -2 gpurun_out/plain_c4.log gpurun_out/ncu_c4.log
python scripts/launch_summary.py gpurun_out/launches_c4.csv
