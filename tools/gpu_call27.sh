mkdir -p gpurun_out
rm -f gpurun_out/variants.txt
for v in base minb1 cbns6 cbseg256; do
  for c in "rmat" "tallskinny" "stencil" "suite-powerlaw-100M"; do
    if [ $v = base ]; then bash tools/quick_bench.sh $c >> gpurun_out/variants.txt 2>&1;
    else MSREP_LIB_VARIANT=tools/libmsrep_$v.so bash tools/quick_bench.sh $c | sed "s/^/$v /" >> gpurun_out/variants.txt 2>&1; fi
  done
done
bash tools/quick_bench.sh suite-powerlaw-100M --format csc >> gpurun_out/variants.txt 2>&1
MSREP_LIB_VARIANT=tools/libmsrep_cbns6.so bash tools/quick_bench.sh suite-powerlaw-100M --format csc | sed "s/^/cbns6 /" >> gpurun_out/variants.txt 2>&1
timeout 600 python tools/spmm_bench.py > gpurun_out/spmm.jsonl 2> gpurun_out/spmm.err
