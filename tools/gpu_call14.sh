mkdir -p gpurun_out
timeout 1200 python tools/imbalance_study.py > gpurun_out/imbalance_study.jsonl 2> gpurun_out/imbalance_study.err
bash tools/suite_sweep.sh
