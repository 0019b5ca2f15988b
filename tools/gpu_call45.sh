mkdir -p gpurun_out
bash tools/gpu_prof.sh banded_csc csc_band_kernel --config suite-banded-100M --format csc
ncu -i gpurun_out/prof_banded_csc.ncu-rep --page raw --csv > gpurun_out/prof_banded_csc_raw.csv 2>&1
