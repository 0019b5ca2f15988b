#!/bin/bash
# tools/gpu_prof.sh TAG KERNEL_REGEX [bench args...]: one ncu --set full capture (2 launches after 3 skipped)
tag=$1; k=$2; shift 2
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o gpurun_out/prof_$tag -f \
  python bench.py --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline "$@" > gpurun_out/ncu_$tag.log 2>&1
echo "ncu $tag rc=$?" >> gpurun_out/ncu_$tag.log
