cd $GRAFT_REPO_ROOT
cd tests && timeout 1200 python -m pytest -x -q test_gpu_fullsize.py -m gpu 2>&1 | tail -5; cd ..
PMMF_B200_TRACE=1 PMMF_B200_SEARCH_TIMING=1 timeout 600 python scripts/configs_full.py c5 --no-pcg > gpurun_out/c5s.log 2> gpurun_out/c5s.err
grep -E "search timing|c=" gpurun_out/c5s.err | head -16
cd tests && timeout 900 python -m pytest -x -q test_gpu_parity.py test_golden.py test_gpu_operator.py -m gpu 2>&1 | tail -2; cd ..
for w in c3 c1; do
timeout 900 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_d$w.json 2> gpurun_out/bench_d$w.err; echo "$w rc=$?"
python -c "
import json
d=json.loads(open('gpurun_out/bench_d$w.json').read().strip().splitlines()[-1])
print(round(d['value']), 'ms/step', round(d['ms_per_step'],1), 'e2e', round(d['e2e']['value']), 'phases', d['phases_ms_last_step'])
"
done
