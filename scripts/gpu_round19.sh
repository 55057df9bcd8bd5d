cd $GRAFT_REPO_ROOT/tests
timeout 900 python -m pytest -x -q test_gpu_parity.py test_golden.py test_dropin.py -m gpu 2>&1 | tail -2
cd ..
timeout 600 python scripts/three_runs.py 3 > gpurun_out/three_m.log 2>&1
grep -E "^run |rror" gpurun_out/three_m.log
sed -n '/^run 1/,$p' gpurun_out/three_m.log | grep -E "stage [0-9]: gram" | head -8
