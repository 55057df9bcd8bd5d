cd $GRAFT_REPO_ROOT
PMMF_B200_TRACE=1 timeout 300 python scripts/one_factorize.py c4 2>&1 | grep -E "clustering|score|stage [1-3]: (gram|apply)|wall|rror" | head -40
timeout 300 python scripts/one_factorize.py c4 > gpurun_out/plain_c4.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4b.csv python scripts/one_factorize.py c4 > gpurun_out/ncu_c4b.log 2>&1
python scripts/launch_summary.py gpurun_out/launches_c4b.csv | head -30
