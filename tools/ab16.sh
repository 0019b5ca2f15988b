mkdir -p gpurun_out/ab
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/ab/pytest_gpu16.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ab/pytest_gpu16.log
O=gpurun_out/ab/ab16.txt
run() { tag=$1; shift; echo "== $tag $*" >> $O; bash tools/quick_bench.sh "$@" >> $O 2>&1; }
for rep in 1 2; do
run ns2 stencil --dtype f32
run ns1 stencil --dtype f32 --sell 3
run ns2-csc stencil --dtype f32 --format csc
run ns1-csc stencil --dtype f32 --format csc --sell 3
run bd-f32 suite-blockdiag-100M --dtype f32
run bd-f32-3 suite-blockdiag-100M --dtype f32 --sell 3
run st64 stencil
done
