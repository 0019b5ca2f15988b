mkdir -p gpurun_out/ab
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/ab/pytest_gpu5.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ab/pytest_gpu5.log
O=gpurun_out/ab/ab5.txt
run() { tag=$1; dir=$2; shift 2; echo "== $tag $*" >> $O; (cd $dir && bash tools/quick_bench.sh "$@") >> $O 2>&1; }
for rep in 1 2; do
  run new . rmat --kernel-times 20
  run gbranch tools/variants/gbranch rmat --kernel-times 20
  run new . stencil --kernel-times 20
  run new . stencil --dtype f32 --kernel-times 20
  run new . random1k --kernel-times 50
  run gbranch tools/variants/gbranch random1k --kernel-times 50
  run new . suite-powerlaw-100M --kernel-times 20
  run new . rmat --format csc --kernel-times 20
done
