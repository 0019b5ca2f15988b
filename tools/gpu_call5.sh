mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
rm -f gpurun_out/qb.txt
for c in "rmat --format csr" "rmat --format coo" "stencil --format coo" "stencil" "stencil --dtype f32" "stencil --format coo --dtype f32" "tallskinny" "random1k"; do bash tools/quick_bench.sh $c >> gpurun_out/qb.txt 2>&1; done
