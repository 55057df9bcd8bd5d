cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --clock-control none --import-source on -k k_score -s 3 -c 1 -o gpurun_out/prof_score2 python scripts/one_factorize.py c4 > gpurun_out/ncu_score2.log 2>&1
tail -2 gpurun_out/ncu_score2.log
