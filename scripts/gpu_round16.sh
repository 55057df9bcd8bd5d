cd $GRAFT_REPO_ROOT
timeout 600 python scripts/three_runs.py 5 > gpurun_out/three_s.log 2>&1
grep -E "^run |rror" gpurun_out/three_s.log
for r in 1 2 3; do echo "-- after run $((r-1))"; awk -v r="run $r" '$0 ~ "^run "{if (index($0, r)==1) exit} f' f=0 gpurun_out/three_s.log >/dev/null; done
awk '/^run /{print; next} /slow alloc|trimmed/{print}' gpurun_out/three_s.log | head -80
