mkdir -p gpurun_out
rm -f gpurun_out/ab.txt
for rep in 1 2; do
for c in "suite-shortwide-100M" "suite-banded-100M" "suite-blockdiag-100M" "rmat" "suite-powerlaw-100M"; do
  bash tools/quick_bench.sh $c | sed "s/^/new /" >> gpurun_out/ab.txt 2>&1
  MSREP_LIB_VARIANT=tools/libmsrep_oldrsum.so bash tools/quick_bench.sh $c | sed "s/^/old /" >> gpurun_out/ab.txt 2>&1
done; done
