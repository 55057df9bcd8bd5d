cd $GRAFT_REPO_ROOT/tests
timeout 120 python -m pytest -x -q test_gpu_parity.py -k "rmat10_m8" 2>&1 | tail -2 || exit 1
timeout 500 python -m pytest -x -q test_gpu_parity.py test_golden.py -m gpu 2>&1 | tail -3
cd ..
PMMF_B200_TRACE=1 timeout 300 python scripts/one_factorize.py c4 2>&1 | grep -E "clustering|score: pool=(5|2|1)[0-9]{5} |wall|rror" | head -12
