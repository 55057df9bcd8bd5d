#!/bin/bash
# Sweep: resident warps of the sparse Gram owner kernel (unused dynamic shared
# memory per 256-thread block caps the blocks per SM, so fewer live
# accumulator columns compete for L2).
tag=${1:-gsweep}; cd $GRAFT_REPO_ROOT; out=gpurun_out/$tag; mkdir -p $out
for sm in 0 45000 75000 110000; do
  PMMF_B200_GRAM_OWNER_SMEM=$sm timeout 900 python bench.py --steps 3 --no-cpu-baseline > $out/bench_$sm.json 2> $out/err_$sm.log
  python -c "import json;d=json.loads(open('$out/bench_$sm.json').read().strip().splitlines()[-1]);print($sm,round(d['ms_per_step'],1),d['phases_ms_last_step']['gram'],d['step_ms'])"
done
