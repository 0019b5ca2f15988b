mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
bash tools/quick_bench.sh rmat --format csc > gpurun_out/rmat_csc_qb.txt 2>&1
bash tools/gpu_prof.sh rmat_csc csc_band_kernel --config rmat --format csc
ncu -i gpurun_out/prof_rmat_csc.ncu-rep --page raw --csv > gpurun_out/prof_rmat_csc_raw.csv 2>&1
