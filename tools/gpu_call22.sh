mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
rm -f gpurun_out/qb.txt
for c in stencil stencil "stencil --format coo" "rmat"; do bash tools/quick_bench.sh $c >> gpurun_out/qb.txt 2>&1; done
timeout 600 python tools/mirror_bench.py > gpurun_out/mirror_bench.jsonl 2> gpurun_out/mirror_bench.err
