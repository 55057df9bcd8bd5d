cd $GRAFT_REPO_ROOT/tests
timeout 300 python -m pytest -x -q test_gpu_parity.py test_golden.py -m gpu 2>&1 | tail -3
cd ..
PMMF_B200_SEARCH_TIMING=1 PMMF_B200_TRACE=1 timeout 120 python scripts/one_factorize.py c2 2>&1 | grep -E "timing|stage 1:|wall" | head -8
PMMF_B200_SEARCH_TIMING=1 PMMF_B200_TRACE=1 timeout 300 python scripts/one_factorize.py c4 2>&1 | grep -E "timing|score|stage [1-3]: (gram|apply)|wall|rror" | head -30
