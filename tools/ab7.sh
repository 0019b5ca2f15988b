mkdir -p gpurun_out/ab
O=gpurun_out/ab/ab7.txt
run() { tag=$1; dir=$2; shift 2; echo "== $tag $*" >> $O; (cd $dir && bash tools/quick_bench.sh "$@") >> $O 2>&1; }
for rep in 1 2; do
  run new . rmat --dtype f32
  run nopdl tools/variants/nopdl rmat --dtype f32
  run new . rmat
  run nopdl tools/variants/nopdl rmat
  run new . stencil
  run nopdl tools/variants/nopdl stencil
  run new . random1k
  run nopdl tools/variants/nopdl random1k
done
