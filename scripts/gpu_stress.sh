cd $GRAFT_REPO_ROOT
cd tests && timeout 900 python -m pytest -x -q test_gpu_parity.py test_golden.py test_gpu_operator.py -m gpu 2>&1 | tail -2; cd ..
for i in 1 2 3; do
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_s$i.json 2> gpurun_out/bench_s$i.err; echo "bench $i rc=$?"; tail -1 gpurun_out/bench_s$i.err | cut -c1-200
python -c "
import json
d=json.loads(open('gpurun_out/bench_s$i.json').read().strip().splitlines()[-1])
print(round(d['value']), 'ms/step', round(d['ms_per_step'],1), [round(x) for x in d['step_ms']], 'e2e', round(d['e2e']['value']), 'phases', d['phases_ms_last_step'])
r=d['roofline']; print(' roofline', {k:round(r[k],3) for k in ('achieved','frac','kernel_ms_total')}, r.get('count_pass'))
" 2>&1 | tail -2
done
