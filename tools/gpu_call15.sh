mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
rm -f gpurun_out/qb.txt
for c in "rmat --format coo_col" "suite-powerlaw-100M --format csc" "suite-banded-100M --format csc" "tallskinny --format coo_col" "stencil --format coo_col" "suite-shortwide-100M --format csc" "tallskinny"; do bash tools/quick_bench.sh $c >> gpurun_out/qb.txt 2>&1; done
