#!/bin/bash
# Hybrid level loop: parity, then config-4 steps for a few thresholds.
tag=${1:-lsweep}; cd $GRAFT_REPO_ROOT; out=gpurun_out/$tag; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "hybrid or level_loop or gram or factorize_matches" > $out/tests.log 2>&1; tail -1 $out/tests.log
for b in 0 256 1024 4096; do
  PMMF_B200_LOOP_BELOW=$b timeout 900 python bench.py --steps 4 --no-cpu-baseline > $out/bench_$b.json 2> $out/err_$b.log
  python -c "import json;d=json.loads(open('$out/bench_$b.json').read().strip().splitlines()[-1]);print($b,round(d['ms_per_step'],1),d['phases_ms_last_step']['apply'],d['step_ms'])"
done
for b in 0 1024; do
  PMMF_B200_LOOP_BELOW=$b timeout 900 python bench.py --workload c5 --steps 4 --no-cpu-baseline > $out/bench_c5_$b.json 2> $out/err_c5_$b.log
  python -c "import json;d=json.loads(open('$out/bench_c5_$b.json').read().strip().splitlines()[-1]);print('c5',$b,round(d['ms_per_step'],1),d['phases_ms_last_step']['apply'],d['step_ms'])"
done
