mkdir -p gpurun_out
timeout 1500 python tools/scaling_projection.py > gpurun_out/scaling_projection.jsonl 2> gpurun_out/scaling_projection.err
