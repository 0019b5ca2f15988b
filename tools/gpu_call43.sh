mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
rm -f gpurun_out/q43.txt
for c in "stencil" "stencil --format coo" "rmat" "rmat --format coo" "suite-blockdiag-100M" "suite-banded-100M"; do bash tools/quick_bench.sh $c >> gpurun_out/q43.txt 2>&1; done
timeout 600 python tools/imbalance_study.py > gpurun_out/imbalance_study.jsonl 2> gpurun_out/imbalance_study.err
