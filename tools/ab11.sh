mkdir -p gpurun_out/ab
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/ab/pytest_gpu11.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ab/pytest_gpu11.log
O=gpurun_out/ab/ab11.txt
run() { tag=$1; shift; echo "== $tag $*" >> $O; bash tools/quick_bench.sh "$@" >> $O 2>&1; }
for rep in 1 2; do
run banded suite-banded-100M
run banded-wide suite-banded-100M --sell 1
run banded-f32 suite-banded-100M --dtype f32
run banded-f32-wide suite-banded-100M --dtype f32 --sell 1
run bd suite-blockdiag-100M
run bd-wide suite-blockdiag-100M --sell 1
run stencil stencil
run rmat rmat
done
