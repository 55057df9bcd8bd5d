cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
for w in c4 c3 c5 c1; do
  timeout 900 python bench.py --workload $w --steps 3 --warmup 3 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; echo "$w rc=$?"
  python -c "
import json,sys
d=json.loads(open('gpurun_out/bench_$w.json').read().strip().splitlines()[-1])
print(d['metric'], round(d['value']), d['unit'], 'ms/step', round(d['ms_per_step'],1), 'e2e', round(d['e2e']['value']), 'phases', d['phases_ms_last_step'])
r=d['roofline']; print(' roofline', r and {k:r[k] for k in ('achieved','peak','frac','unit','kernel_ms_total','launches')}, r and r.get('count_pass'))
print(' cpu', d['cpu_baseline'] and (d['cpu_baseline']['value'], d['cpu_baseline']['sample'][:80]))
print(' apply', d.get('mmf_apply'))
" 2>&1 | tail -5
done
