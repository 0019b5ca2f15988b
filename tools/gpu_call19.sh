mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "mirror" > gpurun_out/pytest_mirror.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_mirror.log
timeout 600 python tools/mirror_bench.py > gpurun_out/mirror_bench.jsonl 2> gpurun_out/mirror_bench.err
