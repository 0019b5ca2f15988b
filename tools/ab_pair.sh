#!/bin/bash
# Same-box A/B of the in-tree build against tools/variants/$1 (default base), alternating runs:
#   tools/ab_pair.sh base "rmat" "suite-powerlaw-100M" ...   (each arg: a quick_bench config + args)
# Output: gpurun_out/ab/pair.txt (kernel ms, frac, clocks per run)
V=${1:-base}; shift
O=gpurun_out/ab; mkdir -p $O
for rep in 1 2; do
  for c in "$@"; do
    echo "== new $c" >> $O/pair.txt
    bash tools/quick_bench.sh $c >> $O/pair.txt 2>&1
    echo "== $V $c" >> $O/pair.txt
    (cd tools/variants/$V && bash tools/quick_bench.sh $c) >> $O/pair.txt 2>&1
  done
done
