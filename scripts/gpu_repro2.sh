cd $GRAFT_REPO_ROOT
for i in 1 2; do
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_r$i.json 2> gpurun_out/bench_r$i.err; echo "bench $i rc=$?"; tail -1 gpurun_out/bench_r$i.err | cut -c1-200
python -c "
import json
d=json.loads(open('gpurun_out/bench_r$i.json').read().strip().splitlines()[-1])
print(round(d['value']), 'ms/step', round(d['ms_per_step'],1), d['step_ms'], 'e2e', round(d['e2e']['value']), 'phases', d['phases_ms_last_step'])
r=d['roofline']; print(' roofline', {k:r[k] for k in ('achieved','frac','kernel_ms_total','launches')}, r.get('count_pass'))
" 2>&1 | tail -2
done
PMMF_B200_PLAN_MAX=0 timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_r3.json 2> gpurun_out/bench_r3.err; echo "bench plan0 rc=$?"; tail -1 gpurun_out/bench_r3.err | cut -c1-200
