cd $GRAFT_REPO_ROOT
python scripts/one_factorize.py c2 > gpurun_out/plain_c2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python scripts/one_factorize.py c2 > gpurun_out/ncu_c2.log 2>&1
python scripts/one_factorize.py s16m512 > gpurun_out/plain_s16.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_s16.csv python scripts/one_factorize.py s16m512 > gpurun_out/ncu_s16.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_search -s 0 -c 1 -o gpurun_out/prof_search_c2 python scripts/one_factorize.py c2 > gpurun_out/ncu_full_c2.log 2>&1
tail -3 gpurun_out/*.log
