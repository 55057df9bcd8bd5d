cd $GRAFT_REPO_ROOT
cd tests && timeout 900 python -m pytest -x -q test_gpu_parity.py test_golden.py test_gpu_operator.py test_dropin.py -m gpu 2>&1 | tail -2; cd ..
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4s.json 2> gpurun_out/bench_c4s.err; echo "rc=$?"
python -c "
import json
d=json.loads(open('gpurun_out/bench_c4s.json').read().strip().splitlines()[-1])
print(round(d['value']), 'ms/step', round(d['ms_per_step'],1), d['step_ms'], 'e2e', round(d['e2e']['value']), 'phases', d['phases_ms_last_step'])
r=d['roofline']; print(' roofline', {k:r[k] for k in ('achieved','frac','kernel_ms_total','launches')}, r.get('count_pass'))
"
PMMF_B200_TRACE=1 timeout 600 python scripts/three_runs.py 2 > gpurun_out/c4v.log 2>&1; grep -E "^run" gpurun_out/c4v.log
sed -n '/^run 0/,$p' gpurun_out/c4v.log | grep -E "batch cols|masses:" | head -8
