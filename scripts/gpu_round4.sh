cd $GRAFT_REPO_ROOT/tests
timeout 120 python -m pytest -x -q test_gpu_parity.py -k "rmat10_m8" 2>&1 | tail -3 || exit 1
timeout 900 python -m pytest -q test_gpu_parity.py test_golden.py test_gpu_operator.py test_errors_gpu.py -m gpu 2>&1 | tail -8
cd ..
PMMF_B200_TRACE=1 timeout 300 python scripts/one_factorize.py c4 2>&1 | grep -E "stage [12]:|wall|Error|rror"
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_r1a.json 2> gpurun_out/bench_r1a.err; tail -c 3000 gpurun_out/bench_r1a.json; tail -5 gpurun_out/bench_r1a.err
