mkdir -p gpurun_out/ab
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/ab/pytest_gpu6.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ab/pytest_gpu6.log
timeout 300 python tools/alloc_bench.py > gpurun_out/ab/alloc_bench.txt 2>&1
O=gpurun_out/ab/ab6.txt
run() { tag=$1; shift; echo "== $tag $*" >> $O; bash tools/quick_bench.sh "$@" >> $O 2>&1; }
run csc-narrow stencil --format csc
run csc-wide stencil --format csc --sell 1
run csc-f32-narrow stencil --format csc --dtype f32
run coo_col stencil --format coo_col
run rmatperm rmatperm --kernel-times 20
run rmatperm-csc rmatperm --format csc
run rmat rmat --kernel-times 20
run f32 rmat --dtype f32
run f32-hot32 rmat --dtype f32 --hot-x 32
run f32-hot48 rmat --dtype f32 --hot-x 48
run pl-f32 suite-powerlaw-100M --dtype f32
run pl-f32-hot32 suite-powerlaw-100M --dtype f32 --hot-x 32
