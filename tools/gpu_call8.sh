mkdir -p gpurun_out
rm -f gpurun_out/qb_var.txt
for v in n3s128 n3s128p180 n2s128 n4s64 n4s128 n2s256; do
  if [ $v = base ]; then unset MSREP_LIB_VARIANT; else export MSREP_LIB_VARIANT=$PWD/tools/libmsrep_$v.so; fi
  echo "== $v" >> gpurun_out/qb_var.txt
  for c in "tallskinny" "tallskinny --dtype f32"; do bash tools/quick_bench.sh $c --steps 50 >> gpurun_out/qb_var.txt 2>&1; done
done
