mkdir -p gpurun_out/ab
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/ab/pytest_gpu15.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ab/pytest_gpu15.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ab/smoke15.log 2>&1; echo "smoke rc=$?" >> gpurun_out/ab/smoke15.log
O=gpurun_out/ab/ab15.txt
run() { tag=$1; shift; echo "== $tag $*" >> $O; bash tools/quick_bench.sh "$@" >> $O 2>&1; }
run rmat rmat --kernel-times 20
run rmatf32 rmat --dtype f32
run pl suite-powerlaw-100M
run banded suite-banded-100M
run bd suite-blockdiag-100M
run stencil stencil
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/ab/bench_driverlike.json 2> gpurun_out/ab/bench_driverlike.err
