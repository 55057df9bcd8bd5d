#!/bin/bash
# Generic check job: GPU suite (or a subset: $TESTS), smoke, and the config-4
# bench line with each rotation-pass driver (persistent level loop / per-level
# launch chain).  Usage: gpurun -- 'bash scripts/gpu_check.sh TAG [TESTS]'
tag=${1:-check}; tests=${2:-tests}
cd $GRAFT_REPO_ROOT; out=gpurun_out/$tag; mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $out/gpu.txt
timeout 2400 python -m pytest $tests -q -x -m gpu > $out/gpu_tests.log 2>&1; echo "gpu tests exit $?" >> $out/gpu_tests.log
tail -3 $out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke exit $?" >> $out/smoke.log
tail -2 $out/smoke.log
for ll in 1 0; do
  PMMF_B200_LEVEL_LOOP=$ll timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $out/bench_c4_ll$ll.json 2> $out/bench_c4_ll$ll.err; echo "bench ll=$ll exit $?"
  python -c "import json;d=json.loads(open('$out/bench_c4_ll$ll.json').read().strip().splitlines()[-1]);print($ll,d['value'],d['ms_per_step'],d['phases_ms_last_step'],d['step_ms'])"
done
