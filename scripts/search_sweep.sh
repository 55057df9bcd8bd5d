# Cluster-search width model sweep on config 4 (search phase per setting).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/sweep
run() {
  echo "== $1" >> gpurun_out/sweep/summary.txt
  env $2 timeout 300 python scripts/stress_repeat.py c4 4 > gpurun_out/sweep/$1.log 2>&1
  tail -4 gpurun_out/sweep/$1.log | cut -c1-110 >> gpurun_out/sweep/summary.txt
}
run default ""
run fit8 "PMMF_B200_SEARCH_A1=3 PMMF_B200_SEARCH_ACL=6.3 PMMF_B200_SEARCH_BETA=0.0055"
run fit16 "PMMF_B200_SEARCH_A1=3 PMMF_B200_SEARCH_ACL=6.3 PMMF_B200_SEARCH_BETA=0.0055 PMMF_B200_SEARCH_CSIZE=16"
run def16 "PMMF_B200_SEARCH_CSIZE=16"
cat gpurun_out/sweep/summary.txt
