cd $GRAFT_REPO_ROOT
echo default; timeout 600 python scripts/repro_c4.py 5 2>&1 | tail -5
echo plan0; PMMF_B200_PLAN_MAX=0 timeout 600 python scripts/repro_c4.py 4 2>&1 | tail -4
echo chunk1024; PMMF_B200_MERGE_CHUNK=1024 timeout 600 python scripts/repro_c4.py 4 2>&1 | tail -4
