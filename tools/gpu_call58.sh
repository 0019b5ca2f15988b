mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
rm -f gpurun_out/bench_lines.jsonl
for c in "--config rmat" "--config rmat --format coo" "--config tallskinny" "--config stencil --format coo" "--config stencil --format csc" "--config stencil --dtype f32" "--config random1k" "--config tallskinny --dtype f32" "--config rmat --format csc"; do
  timeout 600 python bench.py $c --steps 300 --warmup 10 --cpu-seconds 5 >> gpurun_out/bench_lines.jsonl 2>/dev/null
done
STEPS=200 timeout 2400 bash tools/suite_sweep.sh
