mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "suite" > gpurun_out/pytest_suite.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_suite.log
bash tools/suite_sweep.sh
