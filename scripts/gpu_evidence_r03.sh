#!/bin/bash
# Closing evidence (round 2, third session) on one B200: the whole GPU suite and
# smoke, bench lines of every config (GPU arm + reference arm), the config-4
# ncu launch list with per-launch DRAM bytes (write-pass traffic), and
# --set full captures of the longest k_merge2 write pass and count pass, the
# stage-2 scorer, the sparse Gram owner kernel and the MMF stage apply.
tag=${1:-final3}; cd $GRAFT_REPO_ROOT; out=gpurun_out/$tag; mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $out/gpu.txt
timeout 2400 python -m pytest tests -q -m gpu > $out/gpu_tests.log 2>&1; echo "gpu tests exit $?" >> $out/gpu_tests.log
tail -2 $out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke exit $?" >> $out/smoke.log
tail -2 $out/smoke.log
timeout 900 python bench.py --steps 8 --warmup 3 > $out/bench_c4.json 2> $out/bench_c4.err; echo "bench c4 exit $?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $out/bench_ref_c4.json 2> $out/bench_ref_c4.err; echo "ref c4 exit $?"
timeout 1200 python bench.py --workload c5 > $out/bench_c5.json 2> $out/bench_c5.err; echo "bench c5 exit $?"
timeout 900 python bench.py --workload c3 > $out/bench_c3.json 2> $out/bench_c3.err; echo "bench c3 exit $?"
timeout 900 python bench.py --workload c3 --gram dmma --no-cpu-baseline > $out/bench_c3_dmma.json 2> $out/bench_c3_dmma.err; echo "bench c3 dmma exit $?"
timeout 900 python bench.py --workload c1 > $out/bench_c1.json 2> $out/bench_c1.err; echo "bench c1 exit $?"
for f in c4 ref_c4 c5 c3 c3_dmma c1; do
  python -c "import json;d=json.loads(open('$out/bench_$f.json').read().strip().splitlines()[-1]);print('$f',d['value'],d['ms_per_step'],(d.get('roofline') or {}).get('frac'),(d.get('e2e') or {}).get('value'))" 2>/dev/null
done
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $out/launches.csv python bench.py --launch-list > $out/ncu_list.log 2>&1; echo "ncu list exit $?"
python scripts/launch_summary.py $out/launches.csv > $out/launches_summary.txt 2>&1; head -20 $out/launches_summary.txt
python scripts/merge_traffic.py $out/launches.csv $out/merge_traffic_r03.json
for w in 1 0; do
  S=$(python scripts/pick_launch.py $out/launches.csv k_merge2 "k_merge2<$w")
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_merge2 -s $S -c 1 \
    -o $out/merge2_$w python bench.py --launch-list > $out/ncu_merge2_$w.log 2>&1; tail -1 $out/ncu_merge2_$w.log
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_score -s 1 -c 1 \
  -o $out/score python bench.py --launch-list > $out/ncu_score.log 2>&1; tail -1 $out/ncu_score.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gram_owner -c 1 \
  -o $out/gram_owner python bench.py --launch-list > $out/ncu_gram.log 2>&1; tail -1 $out/ncu_gram.log
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_stage_apply_s -c 1 \
  -o $out/stage_apply python scripts/apply_c5.py > $out/ncu_apply.log 2>&1; tail -1 $out/ncu_apply.log
for f in merge2_1 merge2_0 score gram_owner stage_apply; do
  ncu -i $out/$f.ncu-rep --page details --csv > $out/${f}_details.csv 2>/dev/null
done
gzip -f $out/launches.csv
ls -la $out
