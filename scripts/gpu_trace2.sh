#!/bin/bash
# Traced factorizations (sub-phase timings) of config 5 and config 4 after a warm run each.
tag=${1:-tr}; cd $GRAFT_REPO_ROOT; out=gpurun_out/$tag; mkdir -p $out
WARM=2 timeout 600 python scripts/trace_c4.py c5 2> $out/trace_c5.log; tail -1 $out/trace_c5.log
WARM=2 timeout 600 python scripts/trace_c4.py c4 2> $out/trace_c4.log; tail -1 $out/trace_c4.log
