#!/bin/bash
# Small configs with more steps (step distribution): c1 x20, c3 x10, c5 x10.
tag=${1:-small}; cd $GRAFT_REPO_ROOT; out=gpurun_out/$tag; mkdir -p $out
for spec in "c1 20" "c3 10" "c5 10"; do set -- $spec
  timeout 900 python bench.py --workload $1 --steps $2 --warmup 3 --no-cpu-baseline > $out/bench_$1.json 2> $out/bench_$1.err
  python -c "import json;d=json.loads(open('$out/bench_$1.json').read().strip().splitlines()[-1]);print('$1',round(d['value']),[round(x,1) for x in d['step_ms']]);print(d['phases_ms_last_step'])"
done
