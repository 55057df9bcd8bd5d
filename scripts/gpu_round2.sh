cd $GRAFT_REPO_ROOT
(cd tests && timeout 900 python -m pytest -x -q test_gpu_parity.py test_golden.py -m gpu 2>&1 | tail -5)
python scripts/one_factorize.py c2
python scripts/one_factorize.py c2
PMMF_B200_TRACE=1 timeout 900 python scripts/one_factorize.py s18 2>&1 | grep -E "stage 1:|stage 2:|wall"
PMMF_B200_TRACE=1 timeout 900 python scripts/one_factorize.py s19 2>&1 | grep -E "stage 1:|stage 2:|wall|Error"
