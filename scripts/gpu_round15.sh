cd $GRAFT_REPO_ROOT
PMMF_B200_DENSE_DIV=0 timeout 600 python scripts/three_runs.py 3 > gpurun_out/three_t.log 2>&1
grep -E "^run |rror" gpurun_out/three_t.log
sed -n '/^run 1/,$p' gpurun_out/three_t.log | grep -E "reblock" | head -24
