cd $GRAFT_REPO_ROOT
cd tests && timeout 900 python -m pytest -x -q test_gpu_parity.py test_golden.py test_gpu_operator.py -m gpu 2>&1 | tail -2; cd ..
for c in 1024 512 256; do
PMMF_B200_MERGE_CHUNK=$c timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4p$c.json 2> gpurun_out/bench_c4p$c.err; echo "chunk $c rc=$?"
python -c "
import json
d=json.loads(open('gpurun_out/bench_c4p$c.json').read().strip().splitlines()[-1])
print(round(d['value']), 'ms/step', round(d['ms_per_step'],1), 'e2e', round(d['e2e']['value']), 'phases', d['phases_ms_last_step'])
r=d['roofline']; print(' roofline', {k:r[k] for k in ('achieved','frac','kernel_ms_total','launches')}, r.get('count_pass'))
"
done
