#!/bin/bash
# ncu launch list of one config-4 factorization, then --set full captures (with
# source) of the longest k_merge2 write-pass and count-pass launches.
tag=${1:-prof_merge2}; cd $GRAFT_REPO_ROOT; out=gpurun_out/$tag; mkdir -p $out
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv \
  python bench.py --launch-list > $out/ncu.log 2>&1; echo "ncu list exit $?"
python scripts/launch_summary.py $out/launches.csv | head -40 > $out/launches_summary.txt; cat $out/launches_summary.txt
grep -o 'k_merge2<[^>]*>' $out/launches.csv | sort | uniq -c
for w in 1 0; do
  n=$(python scripts/pick_launch.py $out/launches.csv k_merge2 "k_merge2<$w")
  echo "k_merge2 <$w> longest ordinal $n"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_merge2 -s $n -c 1 \
    -o $out/merge2_$w python bench.py --launch-list > $out/ncu_full_$w.log 2>&1; tail -1 $out/ncu_full_$w.log
  ncu -i $out/merge2_$w.ncu-rep --page details --csv > $out/merge2_${w}_details.csv 2>/dev/null
done
gzip -f $out/launches.csv
ls -la $out
