mkdir -p gpurun_out
MSREP_LIB_VARIANT=tools/libmsrep_cbseg256.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_host_resident.py -m gpu -q -k "csc or coo_col or config4 or tallskinny" > gpurun_out/pytest_seg256.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_seg256.log
rm -f gpurun_out/variants2.txt
for v in base cbseg256 seg384 seg192; do
  for c in "tallskinny" "suite-powerlaw-100M --format csc" "suite-shortwide-100M --format csc" "suite-banded-100M --format csc" "tallskinny --dtype f32" "rmat --format coo_col"; do
    if [ $v = base ]; then bash tools/quick_bench.sh $c >> gpurun_out/variants2.txt 2>&1;
    else MSREP_LIB_VARIANT=tools/libmsrep_$v.so bash tools/quick_bench.sh $c | sed "s/^/$v /" >> gpurun_out/variants2.txt 2>&1; fi
  done
done
