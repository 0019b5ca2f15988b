mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
rm -f gpurun_out/q54.txt
for c in "suite-banded-100M" "suite-blockdiag-100M" "rmat" "suite-powerlaw-100M" "suite-shortwide-100M" "stencil" "suite-banded-100M --dtype f32"; do bash tools/quick_bench.sh $c >> gpurun_out/q54.txt 2>&1; done
