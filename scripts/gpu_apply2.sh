cd $GRAFT_REPO_ROOT
cd tests && timeout 900 python -m pytest -x -q test_gpu_operator.py test_golden.py -m gpu 2>&1 | tail -2; cd ..
timeout 900 python scripts/configs_full.py c5 --apply-only > gpurun_out/c5d.log 2>&1; echo rc=$?; grep -E "apply|pcg" gpurun_out/c5d.log | cut -c1-250
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_stage_apply -c 4 -o gpurun_out/prof_apply2 python scripts/configs_full.py c5 --no-pcg --apply-only > gpurun_out/ncu_apply2.log 2>&1; tail -1 gpurun_out/ncu_apply2.log
