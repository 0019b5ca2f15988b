mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -k "csr or coo or rmat or stencil or spmm or sell or host or xload" > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
rm -f gpurun_out/abd.txt
for rep in 1 2; do
for c in "rmat" "suite-banded-100M" "suite-blockdiag-100M" "suite-powerlaw-100M" "suite-shortwide-100M" "stencil --format coo"; do
  bash tools/quick_bench.sh $c | sed "s/^/new /" >> gpurun_out/abd.txt 2>&1
  MSREP_LIB_VARIANT=tools/libmsrep_olddense.so bash tools/quick_bench.sh $c | sed "s/^/old /" >> gpurun_out/abd.txt 2>&1
done; done
