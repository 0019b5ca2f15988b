mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
rm -f gpurun_out/q49.txt
for c in "random1k" "stencil" "rmat"; do bash tools/quick_bench.sh $c >> gpurun_out/q49.txt 2>&1; done
timeout 900 python tools/scaling_projection.py --configs stencil:csr > gpurun_out/scaling_stencil.jsonl 2>&1
