mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
rm -f gpurun_out/bench_lines.jsonl
for c in "--config rmat" "--config rmat --format coo" "--config tallskinny" "--config stencil --format coo" "--config stencil --format csc" "--config stencil --dtype f32" "--config random1k" "--config tallskinny --dtype f32" "--config rmat --format csc"; do
  timeout 600 python bench.py $c --steps 300 --warmup 10 --cpu-seconds 5 >> gpurun_out/bench_lines.jsonl 2>/dev/null
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_stencil.csv python bench.py --steps 50 --warmup 3 --e2e-steps 3 --no-cpu-baseline > gpurun_out/launches_stencil.log 2>&1
bash tools/gpu_prof.sh stencil_rows rows_kernel --config stencil
bash tools/gpu_prof.sh stencil_coo_rows rows_kernel --config stencil --format coo
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
