mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "csc or CSC" > gpurun_out/pytest_csc.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_csc.log
bash tools/quick_bench.sh tallskinny > gpurun_out/qb_ts.txt 2>&1
bash tools/quick_bench.sh tallskinny --dtype f32 >> gpurun_out/qb_ts.txt 2>&1
for v in base ns2 ns2w4 w4 ns3w4; do
  if [ $v = base ]; then unset MSREP_LIB_VARIANT; else export MSREP_LIB_VARIANT=$PWD/tools/libmsrep_$v.so; fi
  echo "== $v" >> gpurun_out/qb_var.txt
  for c in "rmat --format csr" "rmat --format coo" "stencil --format coo" "stencil"; do bash tools/quick_bench.sh $c >> gpurun_out/qb_var.txt 2>&1; done
done
unset MSREP_LIB_VARIANT
bash tools/gpu_prof.sh ts_band csc_band_kernel --config tallskinny
