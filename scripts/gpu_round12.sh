cd $GRAFT_REPO_ROOT/tests
timeout 300 python -m pytest -x -q test_gpu_parity.py -m gpu 2>&1 | tail -2
cd ..
timeout 600 python scripts/three_runs.py 3 > gpurun_out/three.log 2>&1; grep -E "run |apply\.row|overflow|stage 1: (gram|apply)|score: pool=5|rror" gpurun_out/three.log | head -40; tail -3 gpurun_out/three.log
