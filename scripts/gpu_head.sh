#!/bin/bash
# Check job: full GPU suite, smoke, one config-4 bench line.  Usage: gpurun -- 'bash scripts/gpu_head.sh TAG'
tag=${1:-head}
cd $GRAFT_REPO_ROOT; out=gpurun_out/$tag; mkdir -p $out
timeout 2400 python -m pytest tests -q -x -m gpu > $out/gpu_tests.log 2>&1; echo "gpu tests exit $?" >> $out/gpu_tests.log
tail -3 $out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke exit $?" >> $out/smoke.log
tail -2 $out/smoke.log
timeout 900 python bench.py --steps 4 --warmup 3 --no-cpu-baseline > $out/bench_c4.json 2> $out/bench_c4.err; echo "bench exit $?"
python -c "import json;d=json.loads(open('$out/bench_c4.json').read().strip().splitlines()[-1]);r=d['roofline'];print(round(d['value']),round(d['ms_per_step'],1),d['phases_ms_last_step'],[round(x) for x in d['step_ms']],'frac',round(r['frac'],3),'wms',round(r['kernel_ms_total'],1),'cnt',round(r['count_pass']['ms'],1))"
