cd $GRAFT_REPO_ROOT/tests
timeout 120 python -m pytest -x -q test_gpu_parity.py -k "rmat10_m8" 2>&1 | tail -2 || exit 1
timeout 500 python -m pytest -x -q test_gpu_parity.py test_golden.py -m gpu 2>&1 | tail -3
cd ..
timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 1500 gpurun_out/bench.json; tail -3 gpurun_out/bench.err
