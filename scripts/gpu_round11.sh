cd $GRAFT_REPO_ROOT/tests
timeout 120 python -m pytest -x -q test_gpu_parity.py -k "rmat10_m8" 2>&1 | tail -2 || exit 1
timeout 500 python -m pytest -x -q test_gpu_parity.py test_golden.py -m gpu 2>&1 | tail -3
cd ..
timeout 600 python /root/repo/scripts/three_runs.py 2>&1 | grep -E "run |apply\.row|overflow|stage 1: (gram|apply)|score: pool=5" | head -40
