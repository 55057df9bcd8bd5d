#!/bin/bash
# ncu launch list (per-launch device time) of one config-4 factorization.
tag=${1:-launch}; cd $GRAFT_REPO_ROOT; out=gpurun_out/$tag; mkdir -p $out
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv \
  python bench.py --launch-list > $out/ncu.log 2>&1; echo "ncu exit $?"
python scripts/launch_summary.py $out/launches.csv | head -40 > $out/launches_summary.txt; cat $out/launches_summary.txt
gzip -f $out/launches.csv
