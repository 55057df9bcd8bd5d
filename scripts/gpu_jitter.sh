#!/bin/bash
# Step-jitter diagnostic: config-4 bench steps with every instrumented host call
# above 20 ms reported (PMMF_B200_SLOWCALL), with and without the clock sampler.
tag=${1:-jit}; cd $GRAFT_REPO_ROOT; out=gpurun_out/$tag; mkdir -p $out
PMMF_B200_SLOWCALL=20 timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $out/bench_a.json 2> $out/bench_a.err
python -c "import json;d=json.loads(open('$out/bench_a.json').read().strip().splitlines()[-1]);print([round(x) for x in d['step_ms']]);[print(x) for x in d['phases_ms_steps']]"
grep -c "slow call" $out/bench_a.err; grep "slow call" $out/bench_a.err | sort | uniq -c | sort -rn | head -30
nvidia-smi --query-gpu=power.draw,temperature.gpu,clocks.sm,clocks_throttle_reasons.active --format=csv
