#!/bin/bash
# Round-2 evidence: bench lines (config 4 default, config 5 with the CG block,
# config 3), the reference arm, and ncu --set full captures of the clustering
# (k_norms, k_score stage 2) and reblock (k_reblock_fill stage 2) kernels.
tag=${1:-ev2}; cd $GRAFT_REPO_ROOT; out=gpurun_out/$tag; mkdir -p $out
timeout 900 python bench.py > $out/bench_c4.json 2> $out/bench_c4.err; echo "bench c4 exit $?"
timeout 900 python bench.py --workload c5 > $out/bench_c5.json 2> $out/bench_c5.err; echo "bench c5 exit $?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $out/bench_ref_c4.json 2> $out/bench_ref_c4.err; echo "ref exit $?"
for k in k_norms k_score k_reblock_fill; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
    -o $out/$k python bench.py --launch-list > $out/ncu_$k.log 2>&1; tail -1 $out/ncu_$k.log
  ncu -i $out/$k.ncu-rep --page details --csv > $out/${k}_details.csv 2>/dev/null
done
ls -la $out
