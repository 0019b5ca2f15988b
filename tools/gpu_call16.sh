mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "cg" > gpurun_out/pytest_cg.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_cg.log
for f in csr coo csc; do timeout 300 python tools/cg_bench.py --format $f >> gpurun_out/cg_bench.jsonl 2>> gpurun_out/cg_bench.err; done
