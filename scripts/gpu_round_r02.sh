#!/bin/bash
# Iteration job: selected GPU tests, a traced config-4 factorization and the
# config-4 / config-5 bench lines.  Usage: bash scripts/gpu_round_r02.sh TAG "pytest args..."
tag=${1:-it}; shift
cd $GRAFT_REPO_ROOT; out=gpurun_out/$tag; mkdir -p $out
timeout 1800 python -m pytest "$@" -q -x -m gpu > $out/gpu_tests.log 2>&1; echo "gpu tests exit $?" >> $out/gpu_tests.log
tail -3 $out/gpu_tests.log
timeout 600 python scripts/trace_c4.py c4 > $out/trace_c4.log 2>&1; echo "trace exit $?"; tail -1 $out/trace_c4.log
timeout 900 python bench.py --no-cpu-baseline > $out/bench_c4.json 2> $out/bench_c4.err; echo "bench c4 exit $?"
python -c "import json;d=json.loads(open('$out/bench_c4.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['phases_ms_last_step'],d['step_ms'])"
if [ -n "$C5" ]; then
timeout 1200 python bench.py --workload c5 > $out/bench_c5.json 2> $out/bench_c5.err; echo "bench c5 exit $?"
python -c "import json;d=json.loads(open('$out/bench_c5.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['phases_ms_last_step'],json.dumps(d['cg'])[:1500])"
fi
