#!/bin/bash
# One traced config-4 factorization after two warm ones (sub-phase timings), then a bench line.
tag=${1:-tr}; cd $GRAFT_REPO_ROOT; out=gpurun_out/$tag; mkdir -p $out
timeout 600 python scripts/variance_c4.py 2 2> $out/trace.log; grep "===" $out/trace.log
timeout 900 python bench.py --steps 6 --warmup 3 --no-cpu-baseline > $out/bench.json 2> $out/bench.err
python -c "import json;d=json.loads(open('$out/bench.json').read().strip().splitlines()[-1]);print(round(d['value']),[round(x) for x in d['step_ms']]);[print(p) for p in d['phases_ms_steps']]"
