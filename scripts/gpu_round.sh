# one GPU call: parity tests + exploratory timings with stage trace
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.used --format=csv
(cd tests && timeout 900 python -m pytest -x -q test_gpu_operator.py 2>&1 | tail -25)
PMMF_B200_TRACE=1 timeout 900 python scripts/explore.py ${EXPLORE:-c2 s18} 2>&1 | tail -80
