# Round-1 final evidence set (run from the repo root on the GPU box):
#  bench lines for configs 4/3/5/1, the config-4 launch list, write-pass DRAM
#  traffic, one --set full capture each of the longest write pass (config 4),
#  the dense Gram SYRK (config 3) and the MMF apply stage kernel (config 5).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/final
for w in c4 c3 c5 c1; do
  timeout 900 python bench.py --workload $w --steps 3 --warmup 3 > gpurun_out/final/bench_$w.json 2> gpurun_out/final/bench_$w.err; echo "bench $w rc=$?"
done
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/final/bench_ref_c4.json 2>&1; echo "ref rc=$?"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final/launches_r01.csv \
  python bench.py --launch-list > gpurun_out/final/ncu_launches.log 2>&1; echo "launch list rc=$?"
python scripts/launch_summary.py gpurun_out/final/launches_r01.csv > gpurun_out/final/launches_r01_summary.txt
timeout 1500 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -k regex:k_merge_p --csv --log-file gpurun_out/final/merge_traffic_r01.csv python bench.py --launch-list > gpurun_out/final/ncu_traffic.log 2>&1
python scripts/merge_traffic.py gpurun_out/final/merge_traffic_r01.csv gpurun_out/final/merge_traffic_r01.json
SKIP=$(python scripts/pick_launch.py gpurun_out/final/launches_r01.csv k_merge_p "k_merge_p<2, 1>" 2>/dev/null || echo 0)
echo "write-pass capture skip=$SKIP"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_merge_p -s $SKIP -c 1 \
  -o gpurun_out/final/prof_merge_r01 python bench.py --launch-list > gpurun_out/final/ncu_full_merge.log 2>&1; tail -1 gpurun_out/final/ncu_full_merge.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_syrk_seq -c 1 \
  -o gpurun_out/final/prof_syrk_r01 python bench.py --workload c3 --launch-list > gpurun_out/final/ncu_full_syrk.log 2>&1; tail -1 gpurun_out/final/ncu_full_syrk.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stage_apply_s -c 1 \
  -o gpurun_out/final/prof_apply_r01 python scripts/configs_full.py c5 --apply-only --no-pcg > gpurun_out/final/ncu_full_apply.log 2>&1; tail -1 gpurun_out/final/ncu_full_apply.log
head -24 gpurun_out/final/launches_r01_summary.txt; cat gpurun_out/final/merge_traffic_r01.json
