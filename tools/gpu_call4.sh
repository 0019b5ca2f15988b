mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
rm -f gpurun_out/qb_var.txt
for v in base w4 w16; do
  if [ $v = base ]; then unset MSREP_LIB_VARIANT; else export MSREP_LIB_VARIANT=$PWD/tools/libmsrep_$v.so; fi
  echo "== $v" >> gpurun_out/qb_var.txt
  for c in "rmat --format csr" "rmat --format coo" "stencil --format coo" "stencil"; do bash tools/quick_bench.sh $c >> gpurun_out/qb_var.txt 2>&1; done
done
unset MSREP_LIB_VARIANT
bash tools/gpu_prof.sh rmat_csr_reg rows_kernel --config rmat --format csr
