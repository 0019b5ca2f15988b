mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
rm -f gpurun_out/qb_var.txt
for v in base noearly; do
  if [ $v = base ]; then unset MSREP_LIB_VARIANT; else export MSREP_LIB_VARIANT=$PWD/tools/libmsrep_$v.so; fi
  echo "== $v" >> gpurun_out/qb_var.txt
  for c in "stencil --dtype f32" "stencil --format coo --dtype f32" "suite-banded-100M --dtype f32" "suite-blockdiag-100M --dtype f32" "suite-powerlaw-100M --dtype f32" "rmat --dtype f32" "stencil"; do bash tools/quick_bench.sh $c >> gpurun_out/qb_var.txt 2>&1; done
done
