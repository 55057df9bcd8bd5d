cd $GRAFT_REPO_ROOT
timeout 300 python scripts/fp64_peak.py > gpurun_out/fp64_peak.json 2>&1; cat gpurun_out/fp64_peak.json
cd tests && timeout 900 python -m pytest -x -q test_gpu_parity.py -m gpu -k "gram_paths" 2>&1 | tail -3; cd ..
PMMF_B200_TRACE=1 timeout 600 python scripts/configs_full.py c1 c3 > gpurun_out/configs_c13.log 2> gpurun_out/configs_c13.err; echo rc=$?
grep -E "^c[0-9]|phases" gpurun_out/configs_c13.log; grep "gram dense" gpurun_out/configs_c13.err | head -12; tail -3 gpurun_out/configs_c13.err
