mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python tools/host_resident_bench.py --configs stencil:csr,stencil:coo,rmat:csr,rmat:coo,tallskinny:csc > gpurun_out/host_resident.jsonl 2> gpurun_out/host_resident.err
rm -f gpurun_out/xload.txt
for v in base xl1 xl2; do
  for c in "rmat" "tallskinny" "stencil"; do
    if [ $v = base ]; then bash tools/quick_bench.sh $c >> gpurun_out/xload.txt 2>&1;
    else MSREP_LIB_VARIANT=tools/libmsrep_$v.so bash tools/quick_bench.sh $c | sed "s/^/$v /" >> gpurun_out/xload.txt 2>&1; fi
  done
done
