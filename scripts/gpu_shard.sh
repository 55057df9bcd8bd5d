#!/bin/bash
# Sharded factorization on one B200: virtual-rank parity, one-rank NCCL
# exchanges, smoke, and a config-4 bench line (no regression at N=1).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/shard_smi.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_sharded.py -x -q > gpurun_out/shard_tests.log 2>&1
echo "sharded tests exit $?" >> gpurun_out/shard_tests.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "test_factorize_matches_oracle" > gpurun_out/shard_parity.log 2>&1
echo "parity exit $?" >> gpurun_out/shard_parity.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/shard_smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/shard_smoke.log
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/shard_bench_c4.json 2> gpurun_out/shard_bench_c4.err
echo "bench exit $?" >> gpurun_out/shard_bench_c4.err
