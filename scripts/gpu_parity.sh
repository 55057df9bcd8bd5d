set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
cd $GRAFT_REPO_ROOT/tests
timeout 900 python -m pytest -x -q test_gpu_parity.py -k "rmat10_m8 or grid32 or dense256 or diag64 or trivial8" 2>&1 | tail -30
timeout 1200 python -m pytest -q test_gpu_parity.py 2>&1 | tail -40
