cd $GRAFT_REPO_ROOT
timeout 600 python scripts/three_runs.py 2 > gpurun_out/three_m.log 2>&1
grep -E "^run |rror" gpurun_out/three_m.log
sed -n '/^run 0/,$p' gpurun_out/three_m.log | grep -E "gram" | head -16
