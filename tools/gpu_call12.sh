mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "block_split" > gpurun_out/pytest_block.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_block.log
timeout 1200 python tools/imbalance_study.py > gpurun_out/imbalance_study.jsonl 2> gpurun_out/imbalance_study.err
