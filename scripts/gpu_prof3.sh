cd $GRAFT_REPO_ROOT
timeout 120 python scripts/one_factorize.py c2 > gpurun_out/plain_c2b.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_search -s 0 -c 1 -o gpurun_out/prof_search2_c2 python scripts/one_factorize.py c2 > gpurun_out/ncu_search2.log 2>&1
tail -3 gpurun_out/ncu_search2.log
