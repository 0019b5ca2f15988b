mkdir -p gpurun_out/ab
timeout 1500 python -m pytest tests -m gpu -x -q -k "spmm or mm or loopback" > gpurun_out/ab/pytest_gpu10.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ab/pytest_gpu10.log
timeout 600 python tools/spmm_bench.py --config stencil > gpurun_out/ab/spmm.jsonl 2>&1
timeout 600 python tools/spmm_bench.py --config stencil --format coo >> gpurun_out/ab/spmm.jsonl 2>&1
timeout 900 python tools/spmm_bench.py --config rmat >> gpurun_out/ab/spmm.jsonl 2>&1
