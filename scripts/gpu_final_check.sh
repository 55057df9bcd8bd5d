# End-of-round check on a fresh box: the whole GPU suite, smoke, and the
# default bench line (config 4).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/closing
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/closing/gpu_tests.log 2>&1; echo "gpu tests exit $?" >> gpurun_out/closing/gpu_tests.log
tail -3 gpurun_out/closing/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/closing/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/closing/smoke.log
tail -2 gpurun_out/closing/smoke.log
timeout 900 python bench.py > gpurun_out/closing/bench_c4.json 2> gpurun_out/closing/bench_c4.err; echo "bench exit $?"
tail -c 600 gpurun_out/closing/bench_c4.json
