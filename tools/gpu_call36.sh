mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_host_resident.py tests/test_gpu_xload.py -m gpu -q -x -k "csc or coo_col or config4" > gpurun_out/pytest_seg.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_seg.log
rm -f gpurun_out/segq.txt
for c in "rmat --format csc" "rmat --format coo_col" "tallskinny" "stencil --format csc" "suite-banded-100M --format csc" "suite-blockdiag-100M --format csc" "suite-shortwide-100M --format csc" "suite-powerlaw-100M --format csc"; do
  bash tools/quick_bench.sh $c >> gpurun_out/segq.txt 2>&1
done
