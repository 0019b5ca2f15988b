#!/bin/bash
# tools/gpu_check.sh: one gpurun call = GPU tests + smoke + default bench + quick bench lines (e2e shown).
# Everything lands in gpurun_out/check/.
O=gpurun_out/check; mkdir -p $O; rm -f $O/quick.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench_driverlike.json 2> $O/bench_driverlike.err
for c in "rmat --e2e-steps 20" "tallskinny --e2e-steps 10" "stencil --e2e-steps 20" "rmat --format csc --e2e-steps 20"; do
  echo "== $c" >> $O/quick.txt
  timeout 600 python bench.py --config $c --steps 200 --warmup 10 --no-cpu-baseline 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], 'ms', round(d['ms_per_step'],4), 'e2e', d['e2e'])" >> $O/quick.txt 2>&1
done
