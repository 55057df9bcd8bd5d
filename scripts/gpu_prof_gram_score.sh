# ncu --set full captures of the stage-1 sparse Gram kernel and the stage-2
# sparse scorer on config 4 (round-2 targets), summarised under profiles/.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/prof2
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gram_owner -c 1 \
  -o gpurun_out/prof2/gram_owner python bench.py --launch-list > gpurun_out/prof2/ncu_gram.log 2>&1; tail -1 gpurun_out/prof2/ncu_gram.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_score -s 1 -c 1 \
  -o gpurun_out/prof2/score python bench.py --launch-list > gpurun_out/prof2/ncu_score.log 2>&1; tail -1 gpurun_out/prof2/ncu_score.log
for f in gram_owner score; do
  ncu -i gpurun_out/prof2/$f.ncu-rep --page details --csv > gpurun_out/prof2/${f}_details.csv 2>/dev/null
done
ls -la gpurun_out/prof2
