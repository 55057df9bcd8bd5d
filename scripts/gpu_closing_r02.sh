#!/bin/bash
# Closing check of the final code: GPU suite, smoke, bench lines (configs 4, 5, 3 incl. DMMA, 1) and the reference arm.
tag=${1:-closing}; cd $GRAFT_REPO_ROOT; out=gpurun_out/$tag; mkdir -p $out
timeout 2400 python -m pytest tests -q -m gpu > $out/gpu_tests.log 2>&1; echo "gpu tests exit $?" >> $out/gpu_tests.log
tail -2 $out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke exit $?" >> $out/smoke.log; tail -2 $out/smoke.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $out/bench_ref_c4.json 2> $out/bench_ref_c4.err; echo "ref exit $?"
timeout 900 python bench.py > $out/bench_c4.json 2> $out/bench_c4.err; echo "c4 exit $?"
timeout 1200 python bench.py --workload c5 > $out/bench_c5.json 2> $out/bench_c5.err; echo "c5 exit $?"
timeout 900 python bench.py --workload c3 > $out/bench_c3.json 2> $out/bench_c3.err; echo "c3 exit $?"
timeout 900 python bench.py --workload c3 --gram dmma --no-cpu-baseline > $out/bench_c3_dmma.json 2> $out/bench_c3_dmma.err; echo "c3 dmma exit $?"
timeout 900 python bench.py --workload c1 > $out/bench_c1.json 2> $out/bench_c1.err; echo "c1 exit $?"
for f in c4 ref_c4 c5 c3 c3_dmma c1; do
  python -c "import json;d=json.loads(open('$out/bench_$f.json').read().strip().splitlines()[-1]);print('$f',round(d['value']),round(d['ms_per_step'],1),[round(x) for x in d.get('step_ms') or []],(d.get('roofline') or {}).get('frac'))" 2>/dev/null
done
