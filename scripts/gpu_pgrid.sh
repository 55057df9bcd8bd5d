# Merge kernels on a one-wave persistent grid: parity, repeats, bench line.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/pgrid
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_golden.py -q -m gpu -x -k "matches_oracle or small_batches or golden" > gpurun_out/pgrid/tests.log 2>&1; echo "tests exit $?" >> gpurun_out/pgrid/tests.log
tail -2 gpurun_out/pgrid/tests.log
timeout 400 python scripts/stress_repeat.py c4 5 > gpurun_out/pgrid/c4.log 2>&1; tail -5 gpurun_out/pgrid/c4.log | cut -c1-100
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/pgrid/bench_c4.json 2> gpurun_out/pgrid/bench_c4.err
python -c "
import json; d=json.loads(open('gpurun_out/pgrid/bench_c4.json').read().strip().splitlines()[-1]); r=d['roofline']
print(round(d['value']), round(d['ms_per_step'],1), 'write', round(r['kernel_ms_total'],1), round(r['frac'],3), 'count', round(r['count_pass']['ms'],1), d['phases_ms_last_step'], d['step_ms'])"
