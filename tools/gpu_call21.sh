mkdir -p gpurun_out; rm -f gpurun_out/qb_ab.txt
for rep in 1 2 3; do for v in base nomirror; do
  if [ $v = base ]; then unset MSREP_LIB_VARIANT; else export MSREP_LIB_VARIANT=$PWD/tools/libmsrep_$v.so; fi
  echo "== $v" >> gpurun_out/qb_ab.txt; bash tools/quick_bench.sh stencil --steps 2000 >> gpurun_out/qb_ab.txt 2>&1
done; done
