cd $GRAFT_REPO_ROOT
timeout 900 python scripts/level_stats.py c5 2>&1 | tail -8
cd tests && timeout 900 python -m pytest -x -q test_gpu_parity.py -m gpu 2>&1 | tail -2; cd ..
timeout 600 python scripts/three_runs.py 2 > gpurun_out/c4u.log 2>&1; grep -E "^run" gpurun_out/c4u.log
sed -n '/^run 0/,$p' gpurun_out/c4u.log | grep -E "batch cols|masses:" | head -6
