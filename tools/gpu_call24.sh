mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_host_resident.py -x -q > gpurun_out/pytest_hr.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_hr.log
timeout 900 python tools/host_resident_bench.py > gpurun_out/host_resident.jsonl 2> gpurun_out/host_resident.err
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
