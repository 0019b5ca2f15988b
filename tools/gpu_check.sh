#!/bin/bash
# tools/gpu_check.sh: one gpurun call = GPU tests + smoke + default bench + quick bench lines.
# Everything lands in gpurun_out/check/.
O=gpurun_out/check; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err
for c in "rmat --format csc" "rmat --format coo" "rmat --dtype f32" "tallskinny" "tallskinny --dtype f32" "stencil" "stencil --dtype f32" "stencil --format csc"; do
  echo "== $c" >> $O/quick.txt
  bash tools/quick_bench.sh $c >> $O/quick.txt 2>&1
done
