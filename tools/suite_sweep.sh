#!/bin/bash
# tools/suite_sweep.sh: BASELINE config 5 sweep (SuiteSparse-shaped shapes x sizes x formats x dtypes),
# one bench line each -> gpurun_out/suite_sweep.jsonl
mkdir -p gpurun_out
out=gpurun_out/suite_sweep.jsonl; : > $out
run() { timeout 600 python bench.py --steps ${STEPS:-200} --warmup 5 --e2e-steps 3 --no-cpu-baseline "$@" 2>/dev/null | tail -1 >> $out; }
for shape in banded blockdiag powerlaw shortwide; do
  for size in 1M 10M; do run --config suite-$shape-$size; done
  for fmt in csr coo csc; do for dt in f64 f32; do run --config suite-$shape-100M --format $fmt --dtype $dt; done; done
  run --config suite-$shape-100M --format csc --col-layout 0   # pCSC on row bands, for comparison
done
