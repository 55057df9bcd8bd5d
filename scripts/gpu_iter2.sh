#!/bin/bash
# Iteration job: selected GPU tests, optional variance diagnostic, then
# config-4 bench lines (A/B via env).
# Usage: gpurun -- 'bash scripts/gpu_iter2.sh TAG "pytest args" NVAR "ENV=.. ENV=.." ...'
tag=${1:-iter}; tests=$2; nvar=$3; shift 3
cd $GRAFT_REPO_ROOT; out=gpurun_out/$tag; mkdir -p $out
if [ -n "$tests" ]; then
  timeout 1500 python -m pytest $tests -q -x -m gpu > $out/gpu_tests.log 2>&1; echo "gpu tests exit $?" >> $out/gpu_tests.log
  tail -4 $out/gpu_tests.log
fi
if [ "$nvar" != "0" ]; then
  timeout 600 python scripts/variance_c4.py $nvar 2> $out/variance.log; grep "===" $out/variance.log
fi
i=0
for envs in "$@"; do
  i=$((i+1))
  env $envs timeout 900 python bench.py --steps 4 --warmup 3 --no-cpu-baseline > $out/bench_$i.json 2> $out/bench_$i.err; echo "bench [$envs] exit $?"
  python -c "import json;d=json.loads(open('$out/bench_$i.json').read().strip().splitlines()[-1]);r=d['roofline'];print('$envs',round(d['value']),round(d['ms_per_step'],1),d['phases_ms_last_step'],[round(x) for x in d['step_ms']],'frac',round(r['frac'],3),'wms',round(r['kernel_ms_total'],1),'cnt',round(r['count_pass']['ms'],1))"
done
