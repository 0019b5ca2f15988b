mkdir -p gpurun_out
bash tools/gpu_prof.sh rmat_rows rows_kernel --config rmat
ncu -i gpurun_out/prof_rmat_rows.ncu-rep --page raw --csv > gpurun_out/prof_rmat_rows_raw.csv 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_stencil.csv python bench.py --steps 50 --warmup 3 --e2e-steps 3 --no-cpu-baseline > gpurun_out/launches_stencil.log 2>&1
