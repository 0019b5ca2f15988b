mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
timeout 600 python -m pytest tests/test_gpu_xload.py tests/test_gpu_host_resident.py -q -x > gpurun_out/pytest_xload.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_xload.log
rm -f gpurun_out/xauto.txt
for c in "stencil --format coo" "stencil" "rmat" "tallskinny" "suite-banded-100M" "suite-banded-100M --format csc" "suite-blockdiag-100M --format csc" "suite-shortwide-100M --format csc" "suite-shortwide-100M" "suite-powerlaw-100M"; do
  bash tools/quick_bench.sh $c >> gpurun_out/xauto.txt 2>&1
done
