cd $GRAFT_REPO_ROOT
for frac in 0.2 0.06; do
  echo "== frac $frac"
  PMMF_B200_ARENA_FRAC=$frac timeout 600 python scripts/three_runs.py 3 > gpurun_out/three_$frac.log 2>&1
  grep -E "^run |rror|trimmed" gpurun_out/three_$frac.log | head -40
  grep -E "stage 1:|stage 2:|apply\.|overflow" gpurun_out/three_$frac.log | tail -34 | head -22
done
