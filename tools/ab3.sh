mkdir -p gpurun_out/ab
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/ab/pytest_gpu3.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ab/pytest_gpu3.log
O=gpurun_out/ab/ab3.txt
run() { tag=$1; dir=$2; shift 2; echo "== $tag $*" >> $O; (cd $dir && bash tools/quick_bench.sh "$@") >> $O 2>&1; }
for rep in 1 2; do
  run new . rmat --kernel-times 20
  run gbranch tools/variants/gbranch rmat
  run base tools/variants/base rmat
  run new-fused . rmat --fused-fixup 1 --kernel-times 20
  run new . suite-powerlaw-100M
  run gbranch tools/variants/gbranch suite-powerlaw-100M
  run base tools/variants/base suite-powerlaw-100M
  run new . rmat --dtype f32
  run gbranch tools/variants/gbranch rmat --dtype f32
  run base tools/variants/base rmat --dtype f32
  run new-sell2 . stencil --dtype f32
  run new-sell1 . stencil --dtype f32 --sell 1
  run base tools/variants/base stencil --dtype f32
  run new-sell2 . stencil
  run new-sell1 . stencil --sell 1
  run base tools/variants/base stencil
done
