cd $GRAFT_REPO_ROOT
timeout 300 python scripts/one_factorize.py c4 > gpurun_out/plain_c4d.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4d.csv python scripts/one_factorize.py c4 > gpurun_out/ncu_c4d.log 2>&1
tail -2 gpurun_out/plain_c4d.log; python scripts/launch_summary.py gpurun_out/launches_c4d.csv | head -30
