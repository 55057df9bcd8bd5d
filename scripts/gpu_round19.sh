cd $GRAFT_REPO_ROOT/tests
timeout 900 python -m pytest -x -q test_gpu_parity.py test_golden.py test_gpu_operator.py -m gpu 2>&1 | tail -3
cd ..
PMMF_B200_SEARCH_TIMING=1 timeout 600 python scripts/three_runs.py 3 > gpurun_out/three_m.log 2>&1
grep -E "^run |rror" gpurun_out/three_m.log
sed -n '/^run 1/,$p' gpurun_out/three_m.log | grep -E "search timing|c=|score: pool=(1048576|524405)|clustering:" | head -24
