#!/bin/bash
# tools/gpu_check.sh: one gpurun call = build check + GPU tests + smoke + bench lines + ncu launch list
# + one ncu --set full of the dominant kernel. Everything lands in gpurun_out/.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm > gpurun_out/gpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
for c in "rmat --format csr" "rmat --format coo" "tallskinny" "stencil --dtype f32" "stencil --format coo"; do
  n=$(echo $c | tr ' -' '__')
  timeout 600 python bench.py --config $c --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/bench_$n.json 2> gpurun_out/bench_$n.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_stencil.csv \
  python bench.py --steps 50 --warmup 3 --e2e-steps 3 --no-cpu-baseline > gpurun_out/ncu_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sell_kernel -s 5 -c 2 -o gpurun_out/prof_stencil_sell -f \
  python bench.py --steps 10 --warmup 3 --e2e-steps 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
