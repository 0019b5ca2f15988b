mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log

rm -f gpurun_out/qb.txt
for c in "stencil" "stencil --format coo" "rmat --format csr" "tallskinny" "stencil --dtype f32" "random1k" "suite-powerlaw-100M" "suite-blockdiag-100M" "suite-banded-100M"; do bash tools/quick_bench.sh $c >> gpurun_out/qb.txt 2>&1; done
