mkdir -p gpurun_out
MSREP_LIB_VARIANT=tools/libmsrep_fsell.so timeout 1200 ncu --set full --clock-control none -k regex:rows_kernel -s 3 -c 1 -o gpurun_out/prof_fsell -f python bench.py --config rmat --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/ncu_fsell.log 2>&1
ncu -i gpurun_out/prof_fsell.ncu-rep --page details --csv > gpurun_out/prof_fsell_details.csv 2>&1
