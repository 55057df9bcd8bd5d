#!/bin/bash
# Cluster-search corner race fix: repeated full-size factorizations must all
# succeed and be bit-identical; cluster-search parity; shard model.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "cluster_search or matches_oracle" > gpurun_out/race_parity.log 2>&1
echo "parity exit $?" >> gpurun_out/race_parity.log
timeout 600 python scripts/stress_repeat.py c4 14 > gpurun_out/race_c4.log 2>&1
timeout 300 python scripts/stress_repeat.py c5 10 > gpurun_out/race_c5.log 2>&1
timeout 900 python scripts/shard_model.py --workload c4 > gpurun_out/shard_model_c4.json 2> gpurun_out/shard_model_c4.err
timeout 600 python scripts/shard_model.py --workload c5 > gpurun_out/shard_model_c5.json 2> gpurun_out/shard_model_c5.err
