mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "spmm" > gpurun_out/pytest_spmm.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_spmm.log
rm -f gpurun_out/spmm_bench.jsonl
for c in "stencil --format csr" "stencil --format coo" "rmat --format csr"; do timeout 600 python tools/spmm_bench.py --config $c >> gpurun_out/spmm_bench.jsonl 2>> gpurun_out/spmm_bench.err; done
