mkdir -p gpurun_out
rm -f gpurun_out/f32v.txt
for v in base f32m3 f32t512; do
for c in "stencil --dtype f32" "suite-banded-100M --dtype f32" "suite-blockdiag-100M --dtype f32" "rmat --dtype f32" "suite-powerlaw-100M --dtype f32" "suite-shortwide-100M --dtype f32"; do
  if [ $v = base ]; then bash tools/quick_bench.sh $c >> gpurun_out/f32v.txt 2>&1;
  else MSREP_LIB_VARIANT=tools/libmsrep_$v.so bash tools/quick_bench.sh $c | sed "s/^/$v /" >> gpurun_out/f32v.txt 2>&1; fi
done; done
