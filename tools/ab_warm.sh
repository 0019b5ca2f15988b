#!/bin/bash
# A/B of the hot-x size, the warm-x L1 tier and the SEG tile size on R-MAT / power-law (run under gpurun
# after tools/variant.sh t384 "-DMSREP_TILE_NNZ=384").  Output: gpurun_out/ab/warm.txt
O=gpurun_out/ab; mkdir -p $O
for hw in "32 0" "32 16" "32 32" "32 64" "40 0" "40 32" "24 32" "32 128"; do
  set -- $hw
  echo "== rmat hot=$1 warm=$2" >> $O/warm.txt
  bash tools/quick_bench.sh rmat --hot-x $1 --warm-x $2 >> $O/warm.txt 2>&1
done
for w in 0 32; do
  echo "== powerlaw warm=$w" >> $O/warm.txt
  bash tools/quick_bench.sh suite-powerlaw-100M --warm-x $w >> $O/warm.txt 2>&1
done
if [ -d tools/variants/t384 ]; then
  for hw in "32 0" "48 0" "64 0" "48 32"; do
    set -- $hw
    echo "== t384 rmat hot=$1 warm=$2" >> $O/warm.txt
    (cd tools/variants/t384 && bash tools/quick_bench.sh rmat --hot-x $1 --warm-x $2) >> $O/warm.txt 2>&1
  done
fi
