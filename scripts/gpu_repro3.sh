cd $GRAFT_REPO_ROOT
for i in 1 2 3; do
PMMF_B200_PLAN_MAX=0 timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_p$i.json 2> gpurun_out/bench_p$i.err; echo "plan0 bench $i rc=$?"; tail -1 gpurun_out/bench_p$i.err | cut -c1-200
done
for i in 1 2; do
PMMF_B200_ALLOC_CHECK=1 timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_a$i.json 2> gpurun_out/bench_a$i.err; echo "alloccheck bench $i rc=$?"; grep -v "^\s*$" gpurun_out/bench_a$i.err | tail -3 | cut -c1-300
done
