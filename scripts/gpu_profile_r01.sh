# Round-1 profile set (run from the repo root on the GPU box):
#  1. launch list of one bench step (kernel shares of the step),
#  2. DRAM traffic of every rotation write-pass launch (roofline.traffic),
#  3. one --set full capture of a large write-pass launch (stage-1 row pass).
cd $GRAFT_REPO_ROOT
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01.csv \
  python bench.py --launch-list > gpurun_out/ncu_launches.log 2>&1
python scripts/launch_summary.py gpurun_out/launches_r01.csv > gpurun_out/launches_r01_summary.txt
timeout 1500 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -k regex:k_merge_p --csv --log-file gpurun_out/merge_traffic_r01.csv python bench.py --launch-list > gpurun_out/ncu_traffic.log 2>&1
python scripts/merge_traffic.py gpurun_out/merge_traffic_r01.csv gpurun_out/merge_traffic_r01.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_merge_p -s 4338 -c 2 \
  -o gpurun_out/prof_merge_r01 python bench.py --launch-list > gpurun_out/ncu_full.log 2>&1
head -20 gpurun_out/launches_r01_summary.txt; cat gpurun_out/merge_traffic_r01.json; tail -2 gpurun_out/ncu_full.log
