cd $GRAFT_REPO_ROOT/tests
timeout 600 python -m pytest -x -q test_gpu_parity.py -m gpu -k "cluster_search" 2>&1 | tail -3
cd ..
timeout 600 python scripts/three_runs.py 3 > gpurun_out/three_s.log 2>&1
grep -E "^run |rror" gpurun_out/three_s.log
sed -n '/^run 1/,$p' gpurun_out/three_s.log | grep -E "search|slow|trimmed" | head -12 | cut -c1-250
