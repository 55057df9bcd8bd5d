#!/bin/bash
# Owned-column sharding: the sharded GPU tests, the multi-GPU model on
# config 4 and 5, and a 5-step config-4 bench line.
tag=${1:-shard}; cd $GRAFT_REPO_ROOT; out=gpurun_out/$tag; mkdir -p $out
timeout 1800 python -m pytest tests/test_gpu_sharded.py -q -m gpu > $out/gpu_tests.log 2>&1; echo "sharded tests exit $?" >> $out/gpu_tests.log
tail -2 $out/gpu_tests.log
timeout 1800 python scripts/shard_model.py --workload c4 --worlds 2 4 8 > $out/shard_model_c4.json 2> $out/shard_model_c4.err; echo "model c4 exit $?"
python -c "import json;d=json.load(open('$out/shard_model_c4.json'));print(d['one_gpu_wall_ms'],{w:(round(v['modelled_step_ms']),round(v['modelled_speedup'],2),v['bit_identical_to_one_gpu'],round(v['replicated_ms'])) for w,v in d['worlds'].items()})"
timeout 1200 python scripts/shard_model.py --workload c5 --worlds 2 4 8 > $out/shard_model_c5.json 2> $out/shard_model_c5.err; echo "model c5 exit $?"
python -c "import json;d=json.load(open('$out/shard_model_c5.json'));print(d['one_gpu_wall_ms'],{w:(round(v['modelled_step_ms']),round(v['modelled_speedup'],2),v['bit_identical_to_one_gpu'],round(v['replicated_ms'])) for w,v in d['worlds'].items()})"
timeout 900 python bench.py --steps 5 --no-cpu-baseline > $out/bench_c4.json 2> $out/bench_c4.err; echo "bench exit $?"
python -c "import json;d=json.loads(open('$out/bench_c4.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['step_ms'])"
