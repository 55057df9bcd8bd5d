# ncu --set full capture of the longest config-4 write-pass launch with the
# final round-1 code (one-wave persistent grid), summarised under profiles/.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/prof3
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_merge_p -s 4339 -c 1 \
  -o gpurun_out/prof3/merge_r01e python bench.py --launch-list > gpurun_out/prof3/ncu.log 2>&1; tail -1 gpurun_out/prof3/ncu.log
ncu -i gpurun_out/prof3/merge_r01e.ncu-rep --page details --csv > gpurun_out/prof3/merge_r01e_details.csv 2>/dev/null
ls -la gpurun_out/prof3
