mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "csr or coo or rmat or stencil or spmm" > gpurun_out/pytest_rows.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_rows.log
MSREP_LIB_VARIANT=tools/libmsrep_t640.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "csr or coo or rmat or stencil or spmm" > gpurun_out/pytest_t640.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_t640.log
rm -f gpurun_out/variants3.txt
for v in base t640 t768; do
  for c in "rmat" "rmat --format coo" "stencil" "stencil --dtype f32" "rmat --dtype f32" "suite-powerlaw-100M" "suite-shortwide-100M" "suite-banded-100M"; do
    if [ $v = base ]; then bash tools/quick_bench.sh $c >> gpurun_out/variants3.txt 2>&1;
    else MSREP_LIB_VARIANT=tools/libmsrep_$v.so bash tools/quick_bench.sh $c | sed "s/^/$v /" >> gpurun_out/variants3.txt 2>&1; fi
  done
done
MSREP_LIB_VARIANT=tools/libmsrep_t640.so timeout 600 python tools/spmm_bench.py > gpurun_out/spmm_t640.jsonl 2>&1
