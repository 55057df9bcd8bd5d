#!/bin/bash
# gpurun job: a subset of the GPU suite. Usage: bash scripts/gpu_tests.sh TAG "pytest args"
tag=${1:-tests}; shift
cd $GRAFT_REPO_ROOT; out=gpurun_out/$tag; mkdir -p $out
timeout 2400 python -m pytest "$@" -q -m gpu > $out/gpu_tests.log 2>&1; echo "gpu tests exit $?" >> $out/gpu_tests.log
tail -30 $out/gpu_tests.log
