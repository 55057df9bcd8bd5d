#!/bin/bash
# Traced config-4 factorization with each rotation-pass driver.
tag=${1:-trace}; cd $GRAFT_REPO_ROOT; out=gpurun_out/$tag; mkdir -p $out
for ll in 1 0; do
  PMMF_B200_LEVEL_LOOP=$ll timeout 600 python scripts/trace_c4.py c4 > $out/trace_ll$ll.log 2>&1; echo "ll=$ll exit $?"
  tail -2 $out/trace_ll$ll.log
done
