#!/bin/bash
# A/B: 64-row SEG tiles (8 KB less scratch per CTA) with a 48 KiB hot-x cache vs the default 128 rows / 32 KiB
mkdir -p gpurun_out/ab
O=gpurun_out/ab/ab_rows64.txt
run() { tag=$1; dir=$2; shift 2; echo "== $tag $*" >> $O; (cd $dir && bash tools/quick_bench.sh "$@") >> $O 2>&1; }
for rep in 1 2; do
  run base . rmat
  run r64-h48 tools/variants/rows64 rmat --hot-x 48
  run r64-h40 tools/variants/rows64 rmat --hot-x 40
  run pl-base . suite-powerlaw-100M
  run pl-r64-h48 tools/variants/rows64 suite-powerlaw-100M --hot-x 48
done
