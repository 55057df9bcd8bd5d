cd $GRAFT_REPO_ROOT
cd tests && timeout 900 python -m pytest -x -q test_gpu_operator.py test_golden.py -m gpu 2>&1 | tail -2; cd ..
timeout 900 python scripts/configs_full.py c5 --apply-only > gpurun_out/c5c.log 2>&1; echo rc=$?; grep -E "apply|pcg" gpurun_out/c5c.log | cut -c1-250
