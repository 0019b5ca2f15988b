# refresh the committed evidence for the current build: tests, smoke, default bench, launch list,
# ncu --set full of the dominant kernel per key config, suite sweep
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_stencil.csv \
  python bench.py --steps 50 --warmup 3 --e2e-steps 3 --no-cpu-baseline > /dev/null 2>&1
bash tools/gpu_prof.sh stencil_rows rows_kernel
bash tools/gpu_prof.sh stencil_coo_rows rows_kernel --format coo
bash tools/gpu_prof.sh rmat_rows rows_kernel --config rmat
bash tools/gpu_prof.sh ts_csc csc_band_kernel --config tallskinny
bash tools/suite_sweep.sh
