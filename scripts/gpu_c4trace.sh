cd $GRAFT_REPO_ROOT
PMMF_B200_TRACE=1 timeout 900 python scripts/one_factorize.py c4 2>&1 | tail -40
