#!/bin/bash
# One gpurun job: GPU-vs-reference bitwise parity at config 4 (R-MAT scale 14
# and 20 = full) and config 5 (grid 1024^2 = full) with the closing kernels,
# reference under a 185 GB address-space limit (the box has 196 GB, 16 cores).
cd $GRAFT_REPO_ROOT; out=gpurun_out/full_r03; mkdir -p $out
for wl in rmat:14 grid:1024 rmat:20; do
  tag=${wl/:/_}
  python scripts/parity_fullsize.py gpu $wl /tmp/$tag.npz > $out/$tag.gpu.json 2> $out/$tag.gpu.err || continue
  ( ulimit -v 193986560; python scripts/parity_fullsize.py ref $wl /tmp/$tag.npz ) \
      > $out/$tag.ref.json 2> $out/$tag.ref.err
  echo "$wl rc=$?" >> $out/summary.txt
  cat $out/$tag.ref.json >> $out/summary.txt
done
cat $out/summary.txt | cut -c1-400
