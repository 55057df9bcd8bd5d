cd $GRAFT_REPO_ROOT
PMMF_B200_TRACE=1 PMMF_B200_SCORE_TIMING=1 timeout 600 python scripts/one_factorize.py c4 > gpurun_out/sc4.log 2>&1
grep -E "score|clustering" gpurun_out/sc4.log | head -12
