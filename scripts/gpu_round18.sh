cd $GRAFT_REPO_ROOT
PMMF_B200_ALLOC_CHECK=1 timeout 300 python scripts/e2e_repro.py 20 > gpurun_out/e2e.log 2>&1; grep -E "^ok|rror|pmmf\]" gpurun_out/e2e.log | head -20
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 600 gpurun_out/bench.json; tail -3 gpurun_out/bench.err
