#!/bin/bash
# Sweep of the hub-column threshold of the sparse scorer (anchor entries / DIV)
tag=${1:-sweep}; cd $GRAFT_REPO_ROOT; out=gpurun_out/$tag; mkdir -p $out
for div in 4 16 64 256; do
  PMMF_B200_DENSE_DIV=$div timeout 900 python bench.py --steps 3 --no-cpu-baseline > $out/bench_div$div.json 2> $out/err_div$div.log
  python -c "import json;d=json.loads(open('$out/bench_div$div.json').read().strip().splitlines()[-1]);print($div,round(d['ms_per_step'],1),d['phases_ms_last_step']['clustering'],d['step_ms'])"
done
