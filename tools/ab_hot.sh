#!/bin/bash
# A/B of the hot-x cache size inside the 164 KiB carve-out (32 vs 40 KiB), alternating, 3 reps
mkdir -p gpurun_out/ab
O=gpurun_out/ab/ab_hot.txt
run() { tag=$1; shift; echo "== $tag $*" >> $O; bash tools/quick_bench.sh "$@" >> $O 2>&1; }
for rep in 1 2 3; do
  run h32 rmat --hot-x 32
  run h40 rmat --hot-x 40
  run pl-h32 suite-powerlaw-100M --hot-x 32
  run pl-h40 suite-powerlaw-100M --hot-x 40
  run pm-h32 rmatperm --hot-x 32
  run pm-h40 rmatperm --hot-x 40
done
