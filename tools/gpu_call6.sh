mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "csc" > gpurun_out/pytest_csc.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_csc.log
rm -f gpurun_out/qb_var.txt
for v in base e2k6; do
  if [ $v = base ]; then unset MSREP_LIB_VARIANT; else export MSREP_LIB_VARIANT=$PWD/tools/libmsrep_$v.so; fi
  echo "== $v" >> gpurun_out/qb_var.txt
  for c in "tallskinny" "tallskinny --dtype f32"; do bash tools/quick_bench.sh $c >> gpurun_out/qb_var.txt 2>&1; done
done
unset MSREP_LIB_VARIANT
bash tools/gpu_prof.sh ts_band2 csc_band_kernel --config tallskinny
