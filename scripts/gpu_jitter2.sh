#!/bin/bash
# Step-jitter experiment: the same 10 config-4 steps unpinned, pinned to 4 cores, and with spinning syncs.
tag=${1:-jit}; cd $GRAFT_REPO_ROOT; out=gpurun_out/$tag; mkdir -p $out
nproc; cat /sys/fs/cgroup/cpu.max 2>/dev/null; uptime
run() { name=$1; shift; "$@" > $out/$name.json 2> $out/$name.err
  python -c "import json;d=json.loads(open('$out/$name.json').read().strip().splitlines()[-1]);print('$name',[round(x) for x in d['step_ms']])"; }
run plain timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline
run pinned timeout 600 taskset -c 8-11 python bench.py --steps 10 --warmup 3 --no-cpu-baseline
run spin env CUDA_DEVICE_SCHEDULE_SPIN=1 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline
run plain2 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline
uptime
