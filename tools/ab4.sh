mkdir -p gpurun_out/ab
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/ab/pytest_gpu4.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ab/pytest_gpu4.log
O=gpurun_out/ab/ab4.txt
run() { tag=$1; dir=$2; shift 2; echo "== $tag $*" >> $O; (cd $dir && bash tools/quick_bench.sh "$@") >> $O 2>&1; }
for rep in 1 2; do
  run new . rmat --kernel-times 20
  run gbranch tools/variants/gbranch rmat
  run new . suite-powerlaw-100M
  run gbranch tools/variants/gbranch suite-powerlaw-100M
  run new . rmat --dtype f32
  run new . stencil --dtype f32 --kernel-times 20
  run new . stencil --kernel-times 20
  run new . stencil --format coo
  run new . suite-banded-100M
  run new . suite-banded-100M --sell 1
  run new . suite-blockdiag-100M
  run new . suite-blockdiag-100M --sell 1
  run new . tallskinny --kernel-times 10
done
