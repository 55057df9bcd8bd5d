cd $GRAFT_REPO_ROOT
cd tests && timeout 900 python -m pytest -x -q test_gpu_parity.py test_golden.py -m gpu -k "factorize_matches or golden" 2>&1 | tail -2; cd ..
PMMF_B200_TRACE=1 timeout 600 python scripts/three_runs.py 2 > gpurun_out/sc5.log 2>&1
grep -E "^run" gpurun_out/sc5.log; sed -n '/^run 0/,$p' gpurun_out/sc5.log | grep -E "score:|clustering:|repair|pool setup" | head -24
