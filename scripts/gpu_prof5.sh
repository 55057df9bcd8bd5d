cd $GRAFT_REPO_ROOT
timeout 300 python scripts/one_factorize.py c4 > gpurun_out/plain_c4c.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_score -s 3 -c 1 -o gpurun_out/prof_score_c4 python scripts/one_factorize.py c4 > gpurun_out/ncu_score.log 2>&1
tail -3 gpurun_out/ncu_score.log
