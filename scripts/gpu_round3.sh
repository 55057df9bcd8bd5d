cd $GRAFT_REPO_ROOT/tests
timeout 120 python -m pytest -x -q test_gpu_parity.py -k "rmat10_m8" 2>&1 | tail -3 || exit 1
timeout 600 python -m pytest -x -q test_gpu_parity.py test_golden.py test_gpu_operator.py test_errors_gpu.py -m gpu 2>&1 | tail -8
cd ..
timeout 120 python scripts/one_factorize.py c2
timeout 120 python scripts/one_factorize.py c2
PMMF_B200_TRACE=1 timeout 200 python scripts/one_factorize.py s18 2>&1 | grep -E "stage 1:|stage 2:|wall"
PMMF_B200_TRACE=1 timeout 400 python scripts/one_factorize.py c4 2>&1 | grep -E "stage [123]:|wall|Error|rror"
