# Closing evidence with the final round-1 code (one-wave merge grid): bench lines
# for configs 4/3/5/1 and the reference arm, the config-4 ncu launch list and
# write-pass DRAM traffic.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/final3
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > gpurun_out/final3/smi.txt 2>&1
for w in c4 c3 c5 c1; do
  timeout 900 python bench.py --workload $w --steps 3 --warmup 3 > gpurun_out/final3/bench_$w.json 2> gpurun_out/final3/bench_$w.err; echo "bench $w rc=$?"
done
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/final3/bench_ref_c4.json 2>&1; echo "ref rc=$?"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final3/launches_r01e.csv \
  python bench.py --launch-list > gpurun_out/final3/ncu_launches.log 2>&1; echo "launch list rc=$?"
python scripts/launch_summary.py gpurun_out/final3/launches_r01e.csv > gpurun_out/final3/launches_r01e_summary.txt
timeout 1500 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -k regex:k_merge_p --csv --log-file gpurun_out/final3/merge_traffic_r01e.csv python bench.py --launch-list > gpurun_out/final3/ncu_traffic.log 2>&1
python scripts/merge_traffic.py gpurun_out/final3/merge_traffic_r01e.csv gpurun_out/final3/merge_traffic_r01e.json
gzip -f gpurun_out/final3/launches_r01e.csv gpurun_out/final3/merge_traffic_r01e.csv
head -24 gpurun_out/final3/launches_r01e_summary.txt; cat gpurun_out/final3/merge_traffic_r01e.json
