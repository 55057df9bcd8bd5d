cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_merge_p -s 4338 -c 2 -o gpurun_out/prof_merge_big python scripts/one_factorize.py c4 > gpurun_out/ncu_merge.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_merge_p -s 56 -c 2 -o gpurun_out/prof_merge_mid python scripts/one_factorize.py c4 >> gpurun_out/ncu_merge.log 2>&1
tail -3 gpurun_out/ncu_merge.log
