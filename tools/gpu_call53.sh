mkdir -p gpurun_out
bash tools/gpu_prof.sh banded_rows rows_kernel --config suite-banded-100M
ncu -i gpurun_out/prof_banded_rows.ncu-rep --page raw --csv > gpurun_out/prof_banded_rows_raw.csv 2>&1
