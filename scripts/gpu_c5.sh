cd $GRAFT_REPO_ROOT
cd tests && timeout 900 python -m pytest -x -q test_gpu_operator.py test_golden.py -m gpu 2>&1 | tail -3; cd ..
PMMF_B200_TRACE=1 timeout 900 python scripts/configs_full.py c5 --rhs 20 > gpurun_out/configs_c5.log 2> gpurun_out/configs_c5.err; echo rc=$?
tail -14 gpurun_out/configs_c5.log; grep -E "stage [0-9]+: (gram|apply|wall)|gram sparse|gram dense" gpurun_out/configs_c5.err | tail -40
