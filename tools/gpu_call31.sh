mkdir -p gpurun_out
bash tools/gpu_prof.sh rmat_rows rows_kernel --config rmat
ncu -i gpurun_out/prof_rmat_rows.ncu-rep --page raw --csv > gpurun_out/prof_rmat_rows_raw.csv 2>&1
ncu -i gpurun_out/prof_rmat_rows.ncu-rep --page details --csv > gpurun_out/prof_rmat_rows_details.csv 2>&1
bash tools/gpu_prof.sh ts_csc csc_band_kernel --config tallskinny
ncu -i gpurun_out/prof_ts_csc.ncu-rep --page raw --csv > gpurun_out/prof_ts_csc_raw.csv 2>&1
ncu -i gpurun_out/prof_ts_csc.ncu-rep --page details --csv > gpurun_out/prof_ts_csc_details.csv 2>&1
ls -la gpurun_out/
