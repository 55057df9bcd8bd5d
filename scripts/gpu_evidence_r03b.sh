#!/bin/bash
# Closing evidence, second pass (after the host-stall fixes): the whole GPU
# suite and smoke, bench lines of every config (more steps for the small
# ones), the reference arm, and the config-4 ncu launch list with per-launch
# DRAM bytes.  The --set full kernel captures of gpu_evidence_r03.sh stand
# (those kernels did not change).
tag=${1:-final3b}; cd $GRAFT_REPO_ROOT; out=gpurun_out/$tag; mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $out/gpu.txt
timeout 2400 python -m pytest tests -q -m gpu > $out/gpu_tests.log 2>&1; echo "gpu tests exit $?" >> $out/gpu_tests.log
tail -2 $out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke exit $?" >> $out/smoke.log
tail -2 $out/smoke.log
timeout 900 python bench.py --steps 12 --warmup 3 > $out/bench_c4.json 2> $out/bench_c4.err; echo "bench c4 exit $?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $out/bench_ref_c4.json 2> $out/bench_ref_c4.err; echo "ref c4 exit $?"
timeout 1200 python bench.py --workload c5 --steps 10 --warmup 3 > $out/bench_c5.json 2> $out/bench_c5.err; echo "bench c5 exit $?"
timeout 900 python bench.py --workload c3 --steps 10 --warmup 3 > $out/bench_c3.json 2> $out/bench_c3.err; echo "bench c3 exit $?"
timeout 900 python bench.py --workload c3 --gram dmma --steps 10 --warmup 3 --no-cpu-baseline > $out/bench_c3_dmma.json 2> $out/bench_c3_dmma.err; echo "bench c3 dmma exit $?"
timeout 900 python bench.py --workload c1 --steps 20 --warmup 3 > $out/bench_c1.json 2> $out/bench_c1.err; echo "bench c1 exit $?"
for f in c4 ref_c4 c5 c3 c3_dmma c1; do
  python -c "import json;d=json.loads(open('$out/bench_$f.json').read().strip().splitlines()[-1]);print('$f',round(d['value']),round(d['ms_per_step'],1),[round(x) for x in d.get('step_ms',[])],(d.get('roofline') or {}).get('frac'),round((d.get('e2e') or {}).get('value') or 0))" 2>/dev/null
done
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $out/launches.csv python bench.py --launch-list > $out/ncu_list.log 2>&1; echo "ncu list exit $?"
python scripts/launch_summary.py $out/launches.csv > $out/launches_summary.txt 2>&1; head -12 $out/launches_summary.txt
python scripts/merge_traffic.py $out/launches.csv $out/merge_traffic_r03.json
gzip -f $out/launches.csv
