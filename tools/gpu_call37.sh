mkdir -p gpurun_out
rm -f gpurun_out/segr.txt
for v in base sr1000 sr3; do
for c in "rmat --format csc" "suite-banded-100M --format csc" "suite-blockdiag-100M --format csc" "stencil --format csc" "tallskinny"; do
  if [ $v = base ]; then bash tools/quick_bench.sh $c >> gpurun_out/segr.txt 2>&1;
  else MSREP_LIB_VARIANT=tools/libmsrep_$v.so bash tools/quick_bench.sh $c | sed "s/^/$v /" >> gpurun_out/segr.txt 2>&1; fi
done; done
