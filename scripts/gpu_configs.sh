cd $GRAFT_REPO_ROOT
PMMF_B200_TRACE=1 timeout 600 python scripts/configs_full.py c1 c3 > gpurun_out/configs_c13.log 2> gpurun_out/configs_c13.err; echo rc=$?
grep -E "^c[0-9]|phases" gpurun_out/configs_c13.log; tail -3 gpurun_out/configs_c13.err
timeout 900 python scripts/configs_full.py c5 --rhs 20 > gpurun_out/configs_c5.log 2>&1; echo rc=$?
tail -12 gpurun_out/configs_c5.log
